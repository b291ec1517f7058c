// Epilogue store-pattern probe (QKV output 320 x 12288 bf16, 96 CTAs x 4 warps):
//  A: lane = column, 32 tokens per lane (64-B segment per warp store)   [epilogue pattern]
//  B: 16-B vector stores, 8 lanes per token row of 256 B (CTA-wide row)  [staged pattern]
//  D: fully contiguous 16-B stores (same bytes, linear)                  [bandwidth ceiling]
#include <cstdio>
#include <cuda_bf16.h>
#include <cuda_runtime.h>

__global__ void k_store(__nv_bfloat16* out, int ldo, int ntok, unsigned long long* cyc, int mode) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  float v[32];
#pragma unroll
  for (int j = 0; j < 32; ++j) v[j] = threadIdx.x * 0.001f + j;
  unsigned long long t0 = clock64();
  if (mode == 0) {
    const int n = blockIdx.x * 128 + warp * 32 + lane;
    for (int cb = 0; cb < ntok; cb += 32) {
#pragma unroll
      for (int j = 0; j < 32; ++j) out[(size_t)(cb + j) * ldo + n] = __float2bfloat16_rn(v[j] + cb);
    }
  } else if (mode == 1) {
    // per instruction: 128 threads cover 8 token rows x 256 B (16 lanes per row)
    const int t = threadIdx.x;
    for (int m = t / 16; m < ntok; m += 8) {
      uint4 val = make_uint4(m, t, 1, 2);
      *reinterpret_cast<uint4*>(out + (size_t)m * ldo + blockIdx.x * 128 + (t % 16) * 8) = val;
    }
  } else {
    const size_t per_cta = (size_t)ntok * 128;   // elements
    uint4* base = reinterpret_cast<uint4*>(out + blockIdx.x * per_cta);
    for (size_t i = threadIdx.x; i < per_cta / 8; i += 128) base[i] = make_uint4(i, 1, 2, 3);
  }
  unsigned long long t1 = clock64();
  if (lane == 0) cyc[blockIdx.x * 4 + warp] = t1 - t0;
}

int main() {
  const int N = 12288, M = 320, blocks = 96;
  __nv_bfloat16* out;
  unsigned long long* cyc;
  cudaMalloc(&out, (size_t)M * N * 2);
  cudaMalloc(&cyc, blocks * 4 * 8);
  unsigned long long h[blocks * 4];
  const char* names[3] = {"A lane=col 64B/warp-store", "B 16B vec, 256B rows  ", "D contiguous 16B      "};
  for (int mode = 0; mode < 3; ++mode)
    for (int ntok : {32, 320}) {
      for (int it = 0; it < 3; ++it) k_store<<<blocks, 128>>>(out, N, ntok, cyc, mode);
      cudaEvent_t a, b;
      cudaEventCreate(&a); cudaEventCreate(&b);
      cudaEventRecord(a);
      for (int it = 0; it < 10; ++it) k_store<<<blocks, 128>>>(out, N, ntok, cyc, mode);
      cudaEventRecord(b);
      cudaEventSynchronize(b);
      float ms;
      cudaEventElapsedTime(&ms, a, b);
      cudaMemcpy(h, cyc, sizeof h, cudaMemcpyDeviceToHost);
      double s = 0;
      for (int i = 0; i < blocks * 4; ++i) s += h[i];
      const double bytes = (double)blocks * 128 * ntok * 2;
      printf("%s ntok %3d: %6.2f us/launch (%5.0f GB/s), %6.0f cycles/warp\n", names[mode], ntok, ms * 100,
             bytes / (ms * 1e-4) / 1e9, s / (blocks * 4));
    }
  printf("%s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
