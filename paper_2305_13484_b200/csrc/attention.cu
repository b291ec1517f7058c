// K4: masked multi-head decode attention over each row's OWN context.
//
// The fused iteration mixes requests that arrived at different times, so
// every row r attends over keys [0, ctx_r) of its own KV slot (ctx_r = pos+1
// for decode/prefill rows, the stale length for orphan rows).  This is the
// device image of "reads each request's KV at its own step offset"
// (current_iteration per row, reference core.py:85; slot = memory_offset,
// core.py:81).
//
// Flash-decoding split-K: grid (splits, heads, rows); each CTA takes CHUNK
// keys, computes scores with 128-bit K loads (a lane group per key,
// shuffle-reduced), a block softmax, and P.V with 128-bit V loads, then
// either writes the normalised output (1 split) or (max, sum, o) partials
// that k_attn_combine merges.
#include "common.cuh"
#include "kernels.cuh"

namespace fl {

constexpr int ATT_CHUNK = 256;
constexpr int ATT_THREADS = 128;

int attn_max_splits(int S) { return (S + ATT_CHUNK - 1) / ATT_CHUNK; }

template <int X> struct NextPow2 {
  static constexpr int v = X <= 1 ? 1 : X <= 2 ? 2 : X <= 4 ? 4 : X <= 8 ? 8 : X <= 16 ? 16 : 32;
};

int attn_keys_per_split(int row_heads, int S) {
  const int full = attn_max_splits(S);
  int splits = 1;
  if (row_heads < 2 * 148) splits = (2 * 148 + row_heads - 1) / row_heads;
  if (splits > full) splits = full;
  const int keys = (S + splits - 1) / splits;
  return (keys + ATT_CHUNK - 1) / ATT_CHUNK * ATT_CHUNK;
}

template <typename T, int HD>
__global__ void __launch_bounds__(ATT_THREADS) k_attn_split(
    const T* __restrict__ q, const fl_row* __restrict__ rows, const int32_t* __restrict__ row_ctx,
    int Hl, const T* __restrict__ kv_layer, int S, T* __restrict__ out, float* __restrict__ ws_o,
    float* __restrict__ ws_ml, int max_splits, int keys_per_split) {
  pdl_trigger();
  pdl_wait();
  constexpr int VEC = 16 / sizeof(T);          // elements per 16-byte load
  constexpr int NV = HD / VEC;                  // 16-byte vectors per key row
  constexpr int G = NextPow2<NV>::v;            // lanes per key (power of two, <= 32)
  constexpr int PER = (NV + G - 1) / G;         // vectors per lane
  constexpr int KPW = 32 / G;                   // keys per warp per step
  constexpr int NW = ATT_THREADS / 32;
  constexpr int NG = ATT_THREADS / NV > 0 ? ATT_THREADS / NV : 1;   // key groups in P.V

  __shared__ float s_p[ATT_CHUNK];
  __shared__ float s_red[32];
  __shared__ __align__(16) float s_acc[NG][HD];

  const int split = blockIdx.x, h = blockIdx.y, r = blockIdx.z;
  const int ctx = row_ctx[r];
  const int kb0 = split * keys_per_split;
  if (kb0 >= ctx) return;
  const int kb1 = min(ctx, kb0 + keys_per_split);
  const int nsplit = (ctx + keys_per_split - 1) / keys_per_split;
  const int slot = rows[r].slot;
  const int D = Hl * HD;

  const T* Kb = kv_layer + ((static_cast<size_t>(slot) * 2 + 0) * Hl + h) * static_cast<size_t>(S) * HD;
  const T* Vb = kv_layer + ((static_cast<size_t>(slot) * 2 + 1) * Hl + h) * static_cast<size_t>(S) * HD;
  const T* qr = q + static_cast<size_t>(r) * D + h * HD;

  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int g = lane % G;           // lane within key group
  const int kw = lane / G;          // key slot within warp
  const float scale = rsqrtf(static_cast<float>(HD));

  float qv[PER][VEC];
#pragma unroll
  for (int p = 0; p < PER; ++p) {
    const int vi = g + p * G;
    if (vi < NV) {
      load16(qr + vi * VEC, qv[p]);
#pragma unroll
      for (int j = 0; j < VEC; ++j) qv[p][j] *= scale;
    }
  }

  const int vi = threadIdx.x % NV;     // P.V: this thread's 16-byte slice of a V row
  const int kg = threadIdx.x / NV;     // ... and its key group
  float acc[VEC];
#pragma unroll
  for (int j = 0; j < VEC; ++j) acc[j] = 0.f;
  float m_run = -INFINITY, l_run = 0.f;

  for (int c0 = kb0; c0 < kb1; c0 += ATT_CHUNK) {
    const int nk = min(ATT_CHUNK, kb1 - c0);
    // ---- scores of this chunk (lane group per key, 16-byte K loads)
    float local_max = -INFINITY;
    for (int kb = warp * KPW; kb < nk; kb += NW * KPW) {
      const int k = kb + kw;
      float dot = 0.f;
      if (k < nk) {
        const T* kr = Kb + static_cast<size_t>(c0 + k) * HD;
#pragma unroll
        for (int p = 0; p < PER; ++p) {
          const int v2 = g + p * G;
          if (v2 < NV) {
            float kf[VEC];
            uint4 raw = ld_stream16(kr + v2 * VEC);
            if constexpr (sizeof(T) == 4) {
              kf[0] = __uint_as_float(raw.x); kf[1] = __uint_as_float(raw.y);
              kf[2] = __uint_as_float(raw.z); kf[3] = __uint_as_float(raw.w);
            } else {
              const __nv_bfloat162* hh = reinterpret_cast<const __nv_bfloat162*>(&raw);
#pragma unroll
              for (int j = 0; j < 4; ++j) {
                float2 f = __bfloat1622float2(hh[j]);
                kf[2 * j] = f.x; kf[2 * j + 1] = f.y;
              }
            }
#pragma unroll
            for (int j = 0; j < VEC; ++j) dot = fmaf(qv[p][j], kf[j], dot);
          }
        }
      }
#pragma unroll
      for (int o = G / 2; o > 0; o >>= 1) dot += __shfl_xor_sync(0xffffffffu, dot, o);
      if (k < nk && g == 0) {
        s_p[k] = dot;
        local_max = fmaxf(local_max, dot);
      }
    }
    local_max = warp_max(local_max);
    if (lane == 0) s_red[warp] = local_max;
    __syncthreads();
    float m_c = s_red[0];
#pragma unroll
    for (int w = 1; w < NW; ++w) m_c = fmaxf(m_c, s_red[w]);
    const float m_new = fmaxf(m_run, m_c);
    const float rescale = __expf(m_run - m_new);   // 0 on the first chunk
    __syncthreads();
    float psum = 0.f;
    for (int k = threadIdx.x; k < nk; k += ATT_THREADS) {
      const float e = __expf(s_p[k] - m_new);
      s_p[k] = e;
      psum += e;
    }
    const float l_c = block_sum(psum, s_red);   // its __syncthreads publishes s_p
    l_run = l_run * rescale + l_c;
    m_run = m_new;
    // ---- P.V of this chunk (16-byte V loads, NG key groups)
#pragma unroll
    for (int j = 0; j < VEC; ++j) acc[j] *= rescale;
    if (kg < NG) {
      for (int k = kg; k < nk; k += NG) {
        const float pk = s_p[k];
        float vf[VEC];
        uint4 raw = ld_stream16(Vb + static_cast<size_t>(c0 + k) * HD + vi * VEC);
        if constexpr (sizeof(T) == 4) {
          vf[0] = __uint_as_float(raw.x); vf[1] = __uint_as_float(raw.y);
          vf[2] = __uint_as_float(raw.z); vf[3] = __uint_as_float(raw.w);
        } else {
          const __nv_bfloat162* hh = reinterpret_cast<const __nv_bfloat162*>(&raw);
#pragma unroll
          for (int j = 0; j < 4; ++j) {
            float2 f = __bfloat1622float2(hh[j]);
            vf[2 * j] = f.x; vf[2 * j + 1] = f.y;
          }
        }
#pragma unroll
        for (int j = 0; j < VEC; ++j) acc[j] = fmaf(pk, vf[j], acc[j]);
      }
    }
    __syncthreads();   // s_p is rewritten by the next chunk
  }
  if (kg < NG) {
#pragma unroll
    for (int j = 0; j < VEC; ++j) s_acc[kg][vi * VEC + j] = acc[j];
  }
  __syncthreads();
  for (int e = threadIdx.x; e < HD; e += ATT_THREADS) {
    float o = 0.f;
#pragma unroll 4
    for (int gi = 0; gi < NG; ++gi) o += s_acc[gi][e];
    if (nsplit == 1) {
      out[static_cast<size_t>(r) * D + h * HD + e] = from_f<T>(o / l_run);
    } else {
      const size_t w = (static_cast<size_t>(r) * Hl + h) * max_splits + split;
      ws_o[w * HD + e] = o;
      if (e == 0) {
        ws_ml[2 * w] = m_run;
        ws_ml[2 * w + 1] = l_run;
      }
    }
  }
}

template <typename T, int HD>
__global__ void k_attn_combine(const int32_t* __restrict__ row_ctx, int Hl,
                               const float* __restrict__ ws_o, const float* __restrict__ ws_ml,
                               int max_splits, int keys_per_split, T* __restrict__ out) {
  pdl_trigger();
  pdl_wait();
  const int h = blockIdx.x, r = blockIdx.y;
  const int nsplit = (row_ctx[r] + keys_per_split - 1) / keys_per_split;
  if (nsplit <= 1) return;
  const size_t w0 = (static_cast<size_t>(r) * Hl + h) * max_splits;
  float M = -INFINITY;
  for (int s = 0; s < nsplit; ++s) M = fmaxf(M, ws_ml[2 * (w0 + s)]);
  float L = 0.f;
  for (int s = 0; s < nsplit; ++s) L += ws_ml[2 * (w0 + s) + 1] * __expf(ws_ml[2 * (w0 + s)] - M);
  for (int e = threadIdx.x; e < HD; e += blockDim.x) {
    float o = 0.f;
    for (int s = 0; s < nsplit; ++s) o += ws_o[(w0 + s) * HD + e] * __expf(ws_ml[2 * (w0 + s)] - M);
    out[static_cast<size_t>(r) * Hl * HD + h * HD + e] = from_f<T>(o / L);
  }
}

template <typename T, int HD>
static int attn_launch(const void* q, const fl_row* rows, const int32_t* row_ctx, int M, int Hl,
                       const void* kv_layer, int S, int kps, void* out, float* ws_o, float* ws_ml,
                       cudaStream_t s) {
  const int ms = attn_max_splits(S);           // workspace stride (CHUNK-sized splits)
  const int splits = (S + kps - 1) / kps;
  launch_k(k_attn_split<T, HD>, dim3(splits, Hl, M), dim3(ATT_THREADS), 0, s, 1, (const T*)q, rows,
           row_ctx, Hl, (const T*)kv_layer, S, (T*)out, ws_o, ws_ml, ms, kps);
  if (splits > 1) {
    launch_k(k_attn_combine<T, HD>, dim3(Hl, M), dim3(HD < 128 ? HD : 128), 0, s, 1, row_ctx, Hl,
             ws_o, ws_ml, ms, kps, (T*)out);
    return 2;
  }
  return 1;
}

int launch_attention(const void* q, const fl_row* rows, const int32_t* row_ctx, int M, int Hl,
                     int hd, const void* kv_layer, int C, int S, int kps, void* out, float* ws_o,
                     float* ws_ml, int dtype, cudaStream_t s) {
  if (M <= 0) return 0;
#define FL_ATT(HDV)                                                                          \
  case HDV:                                                                                  \
    return dtype == FL_DTYPE_BF16                                                            \
               ? attn_launch<bf16, HDV>(q, rows, row_ctx, M, Hl, kv_layer, S, kps, out, ws_o, \
                                        ws_ml, s)                                            \
               : attn_launch<float, HDV>(q, rows, row_ctx, M, Hl, kv_layer, S, kps, out,      \
                                         ws_o, ws_ml, s);
  switch (hd) {
    FL_ATT(64)
    FL_ATT(96)
    FL_ATT(128)
    FL_ATT(256)
    default: return 0;
  }
#undef FL_ATT
}

}  // namespace fl
