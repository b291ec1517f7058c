// tcgen05 / TMEM / TMA GEMM for the projections of the fused decode step.
#pragma once

#include <cuda.h>
#include <cuda_runtime.h>

#include <cstddef>
#include <cstdint>

#include "kernels.cuh"

namespace fl {

struct TcWorkspace {
  void* base = nullptr;        // caller-owned device scratch
  size_t bytes = 0;
  int num_sms = 148;
};

size_t tc_workspace_bytes(int max_rows, int max_n);
int tc_init(TcWorkspace* ws, void* base, size_t bytes);
void tc_destroy(TcWorkspace* ws);
const char* tc_last_error();
// diagnostics: per-CTA [producer wait, producer total, mma wait, mma total] clocks
void tc_set_debug(unsigned long long* p);

// out[M,N] = X[M,K] . W[N,K]^T (+bias, epilogue), bf16 operands, fp32 accumulate in TMEM.
// Returns 0, or -1 with tc_last_error() set (shape the kernel does not cover).
int gemm_tc(TcWorkspace* ws, const GemmArgs& a, cudaStream_t s);

// Persistent stream-K 2-SM GEMM (gemm_sk.cu) behind gemm_tc;
// workspace = fp32 partial slots + self-resetting flags (zeroed by sk_init).
constexpr int SK_MAX_PAIRS = 80;
constexpr int SK_MAX_SPAN = 512;   // tokens per token tile
size_t sk_workspace_bytes();
int sk_init(void* base, size_t bytes);
cudaError_t sk_rearm(void* base, cudaStream_t s);
int gemm_sk(void* ws, int num_sms, const GemmArgs& a, cudaStream_t s);
const char* sk_last_error();
void sk_set_debug(unsigned long long* p);
void sk_tune(int key, int value);

}  // namespace fl
