// Probe: the HBM weight-stream ceiling for a persistent one-CTA-per-SM kernel.
// Each CTA streams its contiguous share of a 2 GiB buffer (>> L2) with 1-D
// bulk copies of CHUNK bytes into a STAGES-deep mbarrier ring, optionally
// plus XB bytes per chunk from a small L2-resident buffer (the activation
// re-read a GEMM CTA does per K step).  Prints weight GB/s.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o stream_probe stream_probe.cu
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>
#include <cstdint>
#include <cstdio>
#include <cstdlib>

__device__ __forceinline__ uint32_t sa(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void wait(uint64_t* b, uint32_t ph) {
  asm volatile(
      "{\n\t.reg .pred d;\nW_%=:\n\tmbarrier.try_wait.parity.shared::cta.b64 d, [%0], %1;\n\t@!d bra W_%=;\n\t}" ::"r"(
          sa(b)),
      "r"(ph));
}
__device__ __forceinline__ void bulk(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(sa(dst)),
      "l"((uint64_t)src), "r"(bytes), "r"(sa(bar))
      : "memory");
}

// ISSUERS threads each own every ISSUERS-th stage
__global__ void stream(const uint8_t* w, size_t per_cta, int chunk, int stages, const uint8_t* x, int xb,
                       int issuers) {
  extern __shared__ __align__(1024) uint8_t sm[];
  __shared__ __align__(8) uint64_t full[32];
  const int t = threadIdx.x;
  if (t == 0)
    for (int i = 0; i < stages; ++i) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(sa(&full[i])));
  asm volatile("fence.mbarrier_init.release.cluster;");
  __syncthreads();
  if (t >= issuers) return;
  const uint8_t* base = w + per_cta * blockIdx.x;
  const int n = (int)(per_cta / chunk);
  const int slot = chunk + xb;
  for (int it = t; it < n; it += issuers) {
    const int st = it % stages;
    if (it >= stages) wait(&full[st], ((it / stages) - 1) & 1);
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(sa(&full[st])),
                 "r"((uint32_t)slot));
    bulk(sm + (size_t)st * slot, base + (size_t)it * chunk, chunk, &full[st]);
    if (xb) bulk(sm + (size_t)st * slot + chunk, x + ((size_t)it * xb) % (1 << 20), xb, &full[st]);
  }
  for (int it = n - stages > 0 ? n - stages : 0; it < n; ++it)
    if (it % issuers == t) wait(&full[it % stages], (it / stages) & 1);
}

// 2-D tensor-map TMA over a [rows][64] bf16 view (the tiled weight layout:
// 128-byte rows, every box of `box_rows` rows is contiguous), SW128
__device__ unsigned long long g_lat[2];
__device__ unsigned long long g_t[2 * 1024];
__global__ void stream_tma(const __grid_constant__ CUtensorMap map, int rows_per_cta, int box_rows, int stages) {
  unsigned long long t_issue[32], lat = 0, nl = 0;
  extern __shared__ __align__(1024) uint8_t sm_raw[];
  uint8_t* sm = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(sm_raw) + 1023) & ~uintptr_t(1023));
  __shared__ __align__(8) uint64_t full[32];
  if (threadIdx.x != 0) return;
  unsigned long long t0;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
  for (int i = 0; i < stages; ++i) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(sa(&full[i])));
  asm volatile("fence.mbarrier_init.release.cluster;");
  const int chunk = box_rows * 128;
  const int n = rows_per_cta / box_rows;
  const int row0 = blockIdx.x * rows_per_cta;
  for (int it = 0; it < n; ++it) {
    const int st = it % stages;
    if (it >= stages) {
      wait(&full[st], ((it / stages) - 1) & 1);
      lat += clock64() - t_issue[st];
      ++nl;
    }
    t_issue[st] = clock64();
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(sa(&full[st])), "r"((uint32_t)chunk));
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4}], [%2];" ::"r"(
            sa(sm + (size_t)st * chunk)),
        "l"((uint64_t)&map), "r"(sa(&full[st])), "r"(0), "r"(row0 + it * box_rows)
        : "memory");
  }
  for (int it = n - stages > 0 ? n - stages : 0; it < n; ++it) wait(&full[it % stages], (it / stages) & 1);
  atomicAdd(&g_lat[0], lat);
  atomicAdd(&g_lat[1], nl);
  unsigned long long t1;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t1));
  g_t[2 * blockIdx.x] = t0;
  g_t[2 * blockIdx.x + 1] = t1;
}

int main() {
  const size_t total = (size_t)2 << 30;
  uint8_t *w, *x;
  cudaMalloc(&w, total);
  cudaMemset(w, 1, total);
  cudaMalloc(&x, (2 << 20) + 65536);
  cudaMemset(x, 1, (2 << 20) + 65536);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  int nsm = 0;
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
  cudaFuncSetAttribute(stream, cudaFuncAttributeMaxDynamicSharedMemorySize, 220 * 1024);
  struct C { int chunk, stages, xb, issuers, grid_mul; };
  const C cs[] = {
      {16384, 4, 0, 1, 1},  {16384, 8, 0, 1, 1},  {16384, 12, 0, 1, 1}, {32768, 4, 0, 1, 1},
      {32768, 6, 0, 1, 1},  {65536, 3, 0, 1, 1},  {16384, 8, 0, 2, 1},  {16384, 12, 0, 4, 1},
      {16384, 4, 8192, 1, 1}, {16384, 6, 16384, 1, 1}, {16384, 4, 32768, 1, 1}, {32768, 3, 32768, 1, 1},
      {16384, 6, 16384, 2, 1}, {32768, 4, 16384, 2, 1}, {16384, 4, 0, 1, 2}, {16384, 6, 0, 1, 2},
  };
  for (const C& c : cs) {
    const int grid = nsm * c.grid_mul;
    const int smem = c.stages * (c.chunk + c.xb);
    if (smem > 220 * 1024 || (c.grid_mul == 2 && smem > 110 * 1024)) continue;
    const size_t per = (total / grid) / c.chunk * c.chunk;
    stream<<<grid, 128, smem>>>(w, per, c.chunk, c.stages, x, c.xb, c.issuers);
    cudaEventRecord(a);
    const int reps = 5;
    for (int r = 0; r < reps; ++r) stream<<<grid, 128, smem>>>(w, per, c.chunk, c.stages, x, c.xb, c.issuers);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    printf("chunk %6d stages %2d x/chunk %6d issuers %d grid %3d: weights %.0f GB/s (+x %.0f GB/s L2) %s\n",
           c.chunk, c.stages, c.xb, c.issuers, grid, (double)per * grid * reps / (ms * 1e-3) / 1e9,
           (double)per / c.chunk * c.xb * grid * reps / (ms * 1e-3) / 1e9, cudaGetErrorString(cudaGetLastError()));
  }
  // tensor-map TMA over the same bytes viewed as [rows][64] bf16
  PFN_cuTensorMapEncodeTiled_v12000 enc;
  cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", (void**)&enc, cudaEnableDefault, &q);
  cudaFuncSetAttribute(stream_tma, cudaFuncAttributeMaxDynamicSharedMemorySize, 220 * 1024);
  const size_t rows_total = total / 128;
  for (int box : {128, 256}) {
    CUtensorMap map;
    cuuint64_t dims[2] = {64, (cuuint64_t)rows_total}, str[1] = {128};
    cuuint32_t bx[2] = {64, (cuuint32_t)box}, es[2] = {1, 1};
    CUresult r = enc(&map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, w, dims, str, bx, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                     CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) { printf("encode failed %d\n", (int)r); continue; }
    for (int stages : {4, 6, 8}) {
      const int chunk = box * 128;
      const int smem = stages * chunk + 1024;
      if (smem > 220 * 1024) continue;
      const int grid = nsm;
      const int rows_per = (int)((rows_total / grid) / box * box);
      stream_tma<<<grid, 32, smem>>>(map, rows_per, box, stages);
      unsigned long long z[2] = {0, 0};
      cudaMemcpyToSymbol(g_lat, z, sizeof z);
      cudaEventRecord(a);
      const int reps = 5;
      for (int rr = 0; rr < reps; ++rr) stream_tma<<<grid, 32, smem>>>(map, rows_per, box, stages);
      cudaEventRecord(b);
      cudaEventSynchronize(b);
      float ms;
      cudaEventElapsedTime(&ms, a, b);
      unsigned long long l[2];
      cudaMemcpyFromSymbol(l, g_lat, sizeof l);
      printf("TMA 2D box %3d rows (%d KB) stages %d grid %d: %.0f GB/s, issue->full %.0f clk %s\n", box,
             chunk / 1024, stages, grid, (double)rows_per * 128 * grid * reps / (ms * 1e-3) / 1e9,
             l[1] ? (double)l[0] / l[1] : 0.0, cudaGetErrorString(cudaGetLastError()));
      // per-CTA spread of the last launch (one isolated launch)
      stream_tma<<<grid, 32, smem>>>(map, rows_per, box, stages);
      cudaDeviceSynchronize();
      unsigned long long tt[2 * 1024];
      cudaMemcpyFromSymbol(tt, g_t, sizeof(unsigned long long) * 2 * grid);
      unsigned long long s0 = ~0ull, s1 = 0, e0 = ~0ull, e1 = 0;
      for (int i = 0; i < grid; ++i) {
        s0 = tt[2 * i] < s0 ? tt[2 * i] : s0; s1 = tt[2 * i] > s1 ? tt[2 * i] : s1;
        e0 = tt[2 * i + 1] < e0 ? tt[2 * i + 1] : e0; e1 = tt[2 * i + 1] > e1 ? tt[2 * i + 1] : e1;
      }
      printf("   per-CTA: start spread %.1f us, end %.1f .. %.1f us\n", (s1 - s0) / 1e3, (e0 - s0) / 1e3,
             (e1 - s0) / 1e3);
      // same bytes over a short launch (GEMM-sized: 256 MB)
      const int rows_small = (int)(((size_t)256 << 20) / 128 / grid / box * box);
      stream_tma<<<grid, 32, smem>>>(map, rows_small, box, stages);
      cudaDeviceSynchronize();
      cudaEventRecord(a);
      stream_tma<<<grid, 32, smem>>>(map, rows_small, box, stages);
      cudaEventRecord(b);
      cudaEventSynchronize(b);
      cudaEventElapsedTime(&ms, a, b);
      cudaMemcpyFromSymbol(tt, g_t, sizeof(unsigned long long) * 2 * grid);
      s0 = ~0ull; s1 = 0; e0 = ~0ull; e1 = 0;
      for (int i = 0; i < grid; ++i) {
        s0 = tt[2 * i] < s0 ? tt[2 * i] : s0; s1 = tt[2 * i] > s1 ? tt[2 * i] : s1;
        e0 = tt[2 * i + 1] < e0 ? tt[2 * i + 1] : e0; e1 = tt[2 * i + 1] > e1 ? tt[2 * i + 1] : e1;
      }
      printf("   256 MB launch: %.1f us = %.0f GB/s; start spread %.1f us, end %.1f .. %.1f us\n", ms * 1e3,
             (double)rows_small * 128 * grid / (ms * 1e-3) / 1e9, (s1 - s0) / 1e3, (e0 - s0) / 1e3, (e1 - s0) / 1e3);
    }
  }
  return 0;
}
