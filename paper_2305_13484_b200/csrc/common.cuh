// Shared device helpers for the fused decode step (sm_100a).
#pragma once

#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include <utility>

#include "../../include/flover_b200.h"

#define FL_DEV __device__ __forceinline__

namespace fl {

typedef __nv_bfloat16 bf16;

FL_DEV float to_f(float v) { return v; }
FL_DEV float to_f(bf16 v) { return __bfloat162float(v); }
template <typename T> FL_DEV T from_f(float v);
template <> FL_DEV float from_f<float>(float v) { return v; }
template <> FL_DEV bf16 from_f<bf16>(float v) { return __float2bfloat16_rn(v); }

// 16-byte vector of T: 8 bf16 or 4 floats.
template <typename T> struct Vec16 { static constexpr int N = 16 / sizeof(T); };

// Load 16 bytes (N elements of T) and widen to float.
template <typename T>
FL_DEV void load16(const T* __restrict__ p, float* out) {
  uint4 raw = *reinterpret_cast<const uint4*>(p);
  if constexpr (sizeof(T) == 4) {
    out[0] = __uint_as_float(raw.x); out[1] = __uint_as_float(raw.y);
    out[2] = __uint_as_float(raw.z); out[3] = __uint_as_float(raw.w);
  } else {
    const __nv_bfloat162* h = reinterpret_cast<const __nv_bfloat162*>(&raw);
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      float2 f = __bfloat1622float2(h[i]);
      out[2 * i] = f.x; out[2 * i + 1] = f.y;
    }
  }
}

template <typename T>
FL_DEV void store16(T* __restrict__ p, const float* in) {
  uint4 raw;
  if constexpr (sizeof(T) == 4) {
    raw.x = __float_as_uint(in[0]); raw.y = __float_as_uint(in[1]);
    raw.z = __float_as_uint(in[2]); raw.w = __float_as_uint(in[3]);
  } else {
    __nv_bfloat162* h = reinterpret_cast<__nv_bfloat162*>(&raw);
#pragma unroll
    for (int i = 0; i < 4; ++i) h[i] = __floats2bfloat162_rn(in[2 * i], in[2 * i + 1]);
  }
  *reinterpret_cast<uint4*>(p) = raw;
}

// Streaming 16-byte load that does not allocate in L1 (KV / weight streams).
FL_DEV uint4 ld_stream16(const void* p) {
  uint4 r;
  asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];"
               : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w) : "l"(p));
  return r;
}

FL_DEV float warp_sum(float v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

FL_DEV float warp_max(float v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = fmaxf(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}

// Block-wide sum for blockDim.x <= 1024; `red` needs 32 floats of smem.
FL_DEV float block_sum(float v, float* red) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  v = warp_sum(v);
  __syncthreads();
  if (lane == 0) red[warp] = v;
  __syncthreads();
  const int nw = (blockDim.x + 31) >> 5;
  v = (threadIdx.x < nw) ? red[threadIdx.x] : 0.f;
  if (warp == 0) v = warp_sum(v);
  if (threadIdx.x == 0) red[0] = v;
  __syncthreads();
  return red[0];
}

// bf16-output epilogues: tanh.approx.f32 (one MUFU op, |rel err| ~5e-4 in
// tanh, i.e. ~2.5e-4 |x| in GELU -- 16x below the bf16 rounding of the stored
// value); the fp32 paths keep gelu_tanh
FL_DEV float gelu_fast(float x) {
  const float k0 = 0.7978845608028654f, k1 = 0.044715f;
  const float u = k0 * fmaf(k1 * x * x, x, x);
  float t;
  asm("tanh.approx.f32 %0, %1;" : "=f"(t) : "f"(u));
  const float h = 0.5f * x;
  return fmaf(h, t, h);
}

FL_DEV float gelu_tanh(float x) {
  // GPT-2 / GPT-J / NeoX "gelu_new": 0.5 x (1 + tanh(sqrt(2/pi) (x + 0.044715 x^3)))
  // = x / (1 + exp(-2u)), u = sqrt(2/pi) (x + 0.044715 x^3): one SFU exp2 and a
  // fast reciprocal instead of tanhf's ~40-instruction range reduction (the
  // GEMM epilogue evaluates it for every FFN output; |rel err| < 1e-6)
  const float k0 = 0.7978845608028654f, k1 = 0.044715f;
  const float u = k0 * fmaf(k1 * x * x, x, x);
  return __fdividef(x, 1.f + __expf(-2.f * u));
}

// Greedy-token key: max over keys = max logit, ties -> lowest vocab index.
FL_DEV unsigned long long argmax_key(float v, int idx) {
  uint32_t b = __float_as_uint(v);
  b = (b & 0x80000000u) ? ~b : (b | 0x80000000u);
  return (static_cast<unsigned long long>(b) << 32) | (0xFFFFFFFFu - static_cast<uint32_t>(idx));
}
FL_DEV int argmax_key_index(unsigned long long k) {
  return static_cast<int>(0xFFFFFFFFu - static_cast<uint32_t>(k & 0xFFFFFFFFull));
}

// Programmatic dependent launch: every kernel of the step lets its successor
// start its prologue early (launch_dependents) and waits for its
// predecessor's results (wait) before touching them.  Both are no-ops when a
// kernel is launched without the PDL attribute.
FL_DEV void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
FL_DEV void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }

// Row descriptor resolved on the device for every kernel of the step.
struct RowInfo {
  int slot, rid, pos, tok, kind, ctx;
};

// Host: launch with the PDL attribute (and an optional cluster along z).
extern bool g_use_pdl;
template <typename... KArgs, typename... Args>
inline cudaError_t launch_k(void (*k)(KArgs...), dim3 grid, dim3 block, size_t smem,
                            cudaStream_t s, dim3 cluster, Args&&... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute at[2];
  unsigned n = 0;
  if (g_use_pdl) {
    at[n].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[n].val.programmaticStreamSerializationAllowed = 1;
    ++n;
  }
  if (cluster.x * cluster.y * cluster.z > 1) {
    at[n].id = cudaLaunchAttributeClusterDimension;
    at[n].val.clusterDim.x = cluster.x;
    at[n].val.clusterDim.y = cluster.y;
    at[n].val.clusterDim.z = cluster.z;
    ++n;
  }
  cfg.attrs = at;
  cfg.numAttrs = n;
  return cudaLaunchKernelEx(&cfg, k, std::forward<Args>(args)...);
}

}  // namespace fl
