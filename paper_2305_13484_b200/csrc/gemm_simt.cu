// SIMT FFMA GEMM: out[M,N] = X[M,K] . W[N,K]^T (+ bias, epilogue).
//
// The exact-fp32 path (C1 tiny GPT and the fp32 variant of C2) and the
// numerical reference for the tensor-core GEMM.  64x64 output tile per
// 256-thread CTA, 4x4 register micro-tile, K staged through shared memory
// in 32-wide slabs.  The bf16 product path uses gemm_tc.cu (tcgen05).
#include "common.cuh"
#include "kernels.cuh"

namespace fl {

constexpr int SG_BM = 64, SG_BN = 64, SG_BK = 32;

template <typename T>
__global__ void __launch_bounds__(256) k_gemm_simt(const T* __restrict__ X, const T* __restrict__ W,
                                                   const T* __restrict__ bias, void* __restrict__ out,
                                                   int M, int N, int K, int ldx, int ldo, int epi) {
  pdl_trigger();
  pdl_wait();
  __shared__ float sx[SG_BK][SG_BM + 4];
  __shared__ float sw[SG_BK][SG_BN + 4];
  const int m0 = blockIdx.y * SG_BM, n0 = blockIdx.x * SG_BN;
  const int tx = threadIdx.x % 16, ty = threadIdx.x / 16;
  float acc[4][4] = {};
  for (int kk = 0; kk < K; kk += SG_BK) {
    // 64 rows x 32 k per operand = 2048 elements, 8 per thread
    for (int e = threadIdx.x; e < SG_BM * SG_BK; e += 256) {
      const int row = e / SG_BK, kc = e % SG_BK;
      const int gm = m0 + row, gn = n0 + row, gk = kk + kc;
      sx[kc][row] = (gm < M && gk < K) ? to_f(X[static_cast<size_t>(gm) * ldx + gk]) : 0.f;
      sw[kc][row] = (gn < N && gk < K) ? to_f(W[static_cast<size_t>(gn) * K + gk]) : 0.f;
    }
    __syncthreads();
#pragma unroll 8
    for (int k = 0; k < SG_BK; ++k) {
      float a[4], b[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) a[i] = sx[k][ty * 4 + i];
#pragma unroll
      for (int j = 0; j < 4; ++j) b[j] = sw[k][tx * 4 + j];
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) acc[i][j] = fmaf(a[i], b[j], acc[i][j]);
    }
    __syncthreads();
  }
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const int gm = m0 + ty * 4 + i;
    if (gm >= M) continue;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int gn = n0 + tx * 4 + j;
      if (gn >= N) continue;
      float v = acc[i][j] + (bias ? to_f(bias[gn]) : 0.f);
      const size_t o = static_cast<size_t>(gm) * ldo + gn;
      switch (epi) {
        case EPI_STORE: static_cast<T*>(out)[o] = from_f<T>(v); break;
        case EPI_GELU: static_cast<T*>(out)[o] = from_f<T>(gelu_tanh(v)); break;
        case EPI_ACC_F32: static_cast<float*>(out)[o] += v; break;
        default: static_cast<float*>(out)[o] = v; break;
      }
    }
  }
}

void gemm_simt(const GemmArgs& a, cudaStream_t s) {
  if (a.M <= 0 || a.N <= 0) return;
  dim3 grid((a.N + SG_BN - 1) / SG_BN, (a.M + SG_BM - 1) / SG_BM);
  if (a.dtype == FL_DTYPE_BF16)
    launch_k(k_gemm_simt<bf16>, dim3(grid), dim3(256), 0, s, 1, (const bf16*)a.x, (const bf16*)a.w, (const bf16*)a.bias,
                                           a.out, a.M, a.N, a.K, a.ldx, a.ldo, a.epi);
  else
    launch_k(k_gemm_simt<float>, dim3(grid), dim3(256), 0, s, 1, (const float*)a.x, (const float*)a.w,
                                            (const float*)a.bias, a.out, a.M, a.N, a.K, a.ldx,
                                            a.ldo, a.epi);
}

}  // namespace fl
