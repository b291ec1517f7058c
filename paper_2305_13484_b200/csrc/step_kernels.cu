// Row-local kernels of the fused decode step: embedding gather (K1),
// LayerNorm (K2), rotary + KV append (K3 epilogue), greedy argmax and the
// per-request state step (K8/K9 -- the device image of core.record_token,
// reference core.py:108-123).
#include "common.cuh"
#include "kernels.cuh"

namespace fl {

// ---------------------------------------------------------------- K1 embed
template <typename T>
__global__ void k_embed(const fl_row* __restrict__ rows, int n_dec,
                        const int32_t* __restrict__ req_tok, const int32_t* __restrict__ req_pos,
                        int32_t* __restrict__ req_ngen, int R, const T* __restrict__ wte,
                        const T* __restrict__ wpe, int d, float* __restrict__ x,
                        int32_t* __restrict__ row_tok, int32_t* __restrict__ row_pos,
                        int32_t* __restrict__ row_ctx, unsigned long long* __restrict__ keys) {
  pdl_trigger();
  pdl_wait();
  const int r = blockIdx.x;
  const fl_row row = rows[r];
  int tok, pos, ctx;
  if (row.kind == FL_ROW_ORPHAN) {
    ctx = row.ctx > 0 ? row.ctx : 1;
    pos = ctx - 1;
    tok = 0;
  } else {
    const int q = row.rid % R;
    pos = row.pos >= 0 ? row.pos : req_pos[q];
    tok = row.tok >= 0 ? row.tok : req_tok[q];
    ctx = pos + 1;
    // first decode row of a freshly fused request: its generation count starts here
    if (row.kind == FL_ROW_DECODE && row.tok >= 0 && threadIdx.x == 0) req_ngen[q] = 0;
  }
  if (threadIdx.x == 0) {
    row_tok[r] = tok;
    row_pos[r] = pos;
    row_ctx[r] = ctx;
    if (r < n_dec) keys[r] = 0ull;
  }
  constexpr int V = Vec16<T>::N;
  const T* e = wte + static_cast<size_t>(tok) * d;
  const T* p = wpe ? wpe + static_cast<size_t>(pos) * d : nullptr;
  float* xo = x + static_cast<size_t>(r) * d;
  for (int i = threadIdx.x * V; i < d; i += blockDim.x * V) {
    float a[V], b[V];
    load16(e + i, a);
    if (p) {
      load16(p + i, b);
#pragma unroll
      for (int j = 0; j < V; ++j) a[j] += b[j];
    }
#pragma unroll
    for (int j = 0; j < V; j += 4)
      *reinterpret_cast<float4*>(xo + i + j) = make_float4(a[j], a[j + 1], a[j + 2], a[j + 3]);
  }
}

void launch_embed(const fl_row* rows, int n_rows, int n_dec, const int32_t* req_tok,
                  const int32_t* req_pos, int32_t* req_ngen, int R, const void* wte,
                  const void* wpe, int d, int dtype, float* x, int32_t* row_tok, int32_t* row_pos,
                  int32_t* row_ctx, unsigned long long* keys, cudaStream_t s) {
  if (n_rows <= 0) return;
  if (dtype == FL_DTYPE_BF16)
    launch_k(k_embed<bf16>, dim3(n_rows), dim3(128), 0, s, 1, rows, n_dec, req_tok, req_pos,
             req_ngen, R, (const bf16*)wte, (const bf16*)wpe, d, x, row_tok, row_pos, row_ctx, keys);
  else
    launch_k(k_embed<float>, dim3(n_rows), dim3(128), 0, s, 1, rows, n_dec, req_tok, req_pos,
             req_ngen, R, (const float*)wte, (const float*)wpe, d, x, row_tok, row_pos, row_ctx,
             keys);
}

// ---------------------------------------------------------------- K2 LayerNorm
// One CTA per row, values kept in registers (d <= 256 threads * 4 * 8).
template <typename T, int PER>
__global__ void __launch_bounds__(256) k_layernorm(const float* __restrict__ x,
                                                   const T* __restrict__ g,
                                                   const T* __restrict__ b, T* __restrict__ out,
                                                   int d, float eps, const T* __restrict__ g2,
                                                   const T* __restrict__ b2, T* __restrict__ out2) {
  pdl_trigger();
  // gridDim.y == 2: a second (gamma, beta, out) of the same rows (NeoX's LN1
  // and LN2 of one residual in one launch)
  if (blockIdx.y) {
    g = g2;
    b = b2;
    out = out2;
  }
  // gamma / beta are weights (never written by a predecessor): load them
  // before the grid dependency wait, off the critical path
  float gv[PER * 4], bv[PER * 4];
#pragma unroll
  for (int c = 0; c < PER; ++c) {
    const int i = (c * blockDim.x + threadIdx.x) * 4;
    if constexpr (sizeof(T) == 2) {   // 8-byte loads: 4 bf16
      uint2 gr = make_uint2(0u, 0u), br = make_uint2(0u, 0u);
      if (i < d) {
        gr = *reinterpret_cast<const uint2*>(g + i);
        br = *reinterpret_cast<const uint2*>(b + i);
      }
      const __nv_bfloat162* g2 = reinterpret_cast<const __nv_bfloat162*>(&gr);
      const __nv_bfloat162* b2 = reinterpret_cast<const __nv_bfloat162*>(&br);
#pragma unroll
      for (int h2 = 0; h2 < 2; ++h2) {
        const float2 gf = __bfloat1622float2(g2[h2]), bf = __bfloat1622float2(b2[h2]);
        gv[4 * c + 2 * h2] = gf.x;
        gv[4 * c + 2 * h2 + 1] = gf.y;
        bv[4 * c + 2 * h2] = bf.x;
        bv[4 * c + 2 * h2 + 1] = bf.y;
      }
    } else {
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        gv[4 * c + j] = i < d ? to_f(g[i + j]) : 0.f;
        bv[4 * c + j] = i < d ? to_f(b[i + j]) : 0.f;
      }
    }
  }
  pdl_wait();
  __shared__ float red[32];
  const int r = blockIdx.x;
  const float* xr = x + static_cast<size_t>(r) * d;
  float v[PER * 4];
  float s = 0.f;
#pragma unroll
  for (int c = 0; c < PER; ++c) {
    const int i = (c * blockDim.x + threadIdx.x) * 4;
    float4 t = i < d ? *reinterpret_cast<const float4*>(xr + i) : make_float4(0, 0, 0, 0);
    v[4 * c] = t.x; v[4 * c + 1] = t.y; v[4 * c + 2] = t.z; v[4 * c + 3] = t.w;
    s += t.x + t.y + t.z + t.w;
  }
  const float mean = block_sum(s, red) / d;
  float q = 0.f;
#pragma unroll
  for (int c = 0; c < PER; ++c) {
    const int i = (c * blockDim.x + threadIdx.x) * 4;
    if (i < d) {
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const float t = v[4 * c + j] - mean;
        q += t * t;
      }
    }
  }
  const float rstd = rsqrtf(block_sum(q, red) / d + eps);
  T* o = out + static_cast<size_t>(r) * d;
#pragma unroll
  for (int c = 0; c < PER; ++c) {
    const int i = (c * blockDim.x + threadIdx.x) * 4;
    if (i < d) {
      if constexpr (sizeof(T) == 2) {
        // 8-byte output stores (4 bf16 per thread)
        __nv_bfloat162 y[2];
#pragma unroll
        for (int h2 = 0; h2 < 2; ++h2)
          y[h2] = __floats2bfloat162_rn((v[4 * c + 2 * h2] - mean) * rstd * gv[4 * c + 2 * h2] + bv[4 * c + 2 * h2],
                                        (v[4 * c + 2 * h2 + 1] - mean) * rstd * gv[4 * c + 2 * h2 + 1] +
                                            bv[4 * c + 2 * h2 + 1]);
        *reinterpret_cast<uint2*>(o + i) = *reinterpret_cast<const uint2*>(y);
      } else {
#pragma unroll
        for (int j = 0; j < 4; ++j)
          o[i + j] = from_f<T>((v[4 * c + j] - mean) * rstd * gv[4 * c + j] + bv[4 * c + j]);
      }
    }
  }
}

template <typename T>
static void ln_dispatch(const float* x, const void* g, const void* b, void* out, int M, int d,
                        float eps, cudaStream_t s, const void* g2 = nullptr, const void* b2 = nullptr,
                        void* out2 = nullptr) {
  const int per = (d + 1023) / 1024;  // float4 chunks per thread at 256 threads
  const T* G = (const T*)g;
  const T* B = (const T*)b;
  T* O = (T*)out;
  const T* G2 = (const T*)g2;
  const T* B2 = (const T*)b2;
  T* O2 = (T*)out2;
  const dim3 grid(M, out2 ? 2 : 1);
#define FL_LN(P) launch_k(k_layernorm<T, P>, grid, dim3(256), 0, s, 1, x, G, B, O, d, eps, G2, B2, O2)
  switch (per) {
    case 1: FL_LN(1); break;
    case 2: FL_LN(2); break;
    case 3: FL_LN(3); break;
    case 4: FL_LN(4); break;
    case 5: case 6: FL_LN(6); break;
    default: FL_LN(8); break;
  }
#undef FL_LN
}

void launch_layernorm(const float* x, const void* g, const void* b, void* out, int M, int d,
                      float eps, int dtype, cudaStream_t s) {
  if (M <= 0) return;
  if (dtype == FL_DTYPE_BF16) ln_dispatch<bf16>(x, g, b, out, M, d, eps, s);
  else ln_dispatch<float>(x, g, b, out, M, d, eps, s);
}

void launch_layernorm2(const float* x, const void* g, const void* b, void* out, const void* g2,
                       const void* b2, void* out2, int M, int d, float eps, int dtype, cudaStream_t s) {
  if (M <= 0) return;
  if (dtype == FL_DTYPE_BF16) ln_dispatch<bf16>(x, g, b, out, M, d, eps, s, g2, b2, out2);
  else ln_dispatch<float>(x, g, b, out, M, d, eps, s, g2, b2, out2);
}

// ---------------------------------------------------------------- residual add
template <typename T>
__global__ void k_add_partial(float* __restrict__ x, const float* __restrict__ y,
                              const T* __restrict__ b1, const T* __restrict__ b2, int M, int d) {
  pdl_trigger();
  pdl_wait();
  const size_t n = static_cast<size_t>(M) * d;
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n;
       i += (size_t)gridDim.x * blockDim.x) {
    const int c = static_cast<int>(i % d);
    float v = x[i] + y[i];
    if (b1) v += to_f(b1[c]);
    if (b2) v += to_f(b2[c]);
    x[i] = v;
  }
}

void launch_add_partial(float* x, const float* y, const void* b1, const void* b2, int M, int d,
                        int dtype, cudaStream_t s) {
  if (M <= 0) return;
  const size_t n = (size_t)M * d;
  const int grid = (int)((n + 255) / 256 < 148 * 8 ? (n + 255) / 256 : 148 * 8);
  if (dtype == FL_DTYPE_BF16)
    launch_k(k_add_partial<bf16>, dim3(grid), dim3(256), 0, s, 1, x, y, (const bf16*)b1, (const bf16*)b2, M, d);
  else
    launch_k(k_add_partial<float>, dim3(grid), dim3(256), 0, s, 1, x, y, (const float*)b1, (const float*)b2, M, d);
}

// ---------------------------------------------------------------- rotary + KV append
// grid (M, Hl), block hd threads: thread i owns element i of q, k and v.
template <typename T>
__global__ void k_rope_append(const T* __restrict__ qkv, const fl_row* __restrict__ rows,
                              const int32_t* __restrict__ row_pos, int Hl, int hd, int rot,
                              int family, T* __restrict__ kv_layer, int C, int S,
                              T* __restrict__ qout, int ldq) {
  pdl_trigger();
  pdl_wait();
  const int r = blockIdx.x, h = blockIdx.y, i = threadIdx.x;
  const int D = Hl * hd;
  const T* base = qkv + static_cast<size_t>(r) * ldq + h * hd;
  float q = to_f(base[i]);
  float k = to_f(base[D + i]);
  const float v = to_f(base[2 * D + i]);
  const int pos = row_pos[r];
  if (rot > 0 && i < rot) {
    // pair partner and frequency index: GPT-J interleaves (2j, 2j+1);
    // NeoX rotates halves (j, j + rot/2).  inv_freq_j = 10000^(-2j/rot).
    int j, partner;
    float sign;
    if (family == FL_FAMILY_GPTJ) {
      j = i >> 1;
      partner = i ^ 1;
      sign = (i & 1) ? 1.f : -1.f;
    } else {
      const int half = rot >> 1;
      j = i < half ? i : i - half;
      partner = i < half ? i + half : i - half;
      sign = i < half ? -1.f : 1.f;
    }
    const float inv_freq = exp2f(-(2.f * j / rot) * 13.287712379549449f);  // log2(10000)
    float sn, cs;
    sincosf(static_cast<float>(pos) * inv_freq, &sn, &cs);
    const float qp = to_f(base[partner]);
    const float kp = to_f(base[D + partner]);
    q = q * cs + sign * qp * sn;
    k = k * cs + sign * kp * sn;
  }
  qout[static_cast<size_t>(r) * D + h * hd + i] = from_f<T>(q);
  const fl_row row = rows[r];
  if (row.kind != FL_ROW_ORPHAN) {
    const size_t kb = ((static_cast<size_t>(row.slot) * 2 + 0) * Hl + h) * S + pos;
    const size_t vb = ((static_cast<size_t>(row.slot) * 2 + 1) * Hl + h) * S + pos;
    kv_layer[kb * hd + i] = from_f<T>(k);
    kv_layer[vb * hd + i] = from_f<T>(v);
  }
}

// sin/cos of the rotary angle pos * 10000^(-2j/rot): the fp32 angle (as the
// precise path forms it) reduced to [-pi, pi] with a two-constant Cody-Waite
// step, then the SFU sincos -- |error| ~1e-6 against sincosf, which spends
// hundreds of instructions per call on its general range reduction
FL_DEV void rope_sincos(float pos, int j, int rot, float* sn, float* cs) {
  const float x = pos * exp2f(-(2.f * j / rot) * 13.287712379549449f);   // log2(10000)
  const float kq = rintf(x * 0.15915494309189535f);
  float rr = fmaf(-kq, 6.28318548202514648f, x);       // 2pi, fp32 head
  rr = fmaf(-kq, -1.7484556e-07f, rr);                  // 2pi - head
  __sincosf(rr, sn, cs);
}

// bf16 variant: one thread per 16-byte vector (8 elements) of q, k and v --
// 16-byte loads and stores instead of 2-byte ones.  GPT-J's interleaved pairs
// (2j, 2j+1) sit inside one vector; NeoX's rotate-half partner (i +- rot/2) is
// read element-wise from the (L1-resident) row.
__global__ void __launch_bounds__(256) k_rope_append_v(const bf16* __restrict__ qkv,
                                                      const fl_row* __restrict__ rows,
                                                      const int32_t* __restrict__ row_pos, int Hl,
                                                      int hd, int rot, int family,
                                                      bf16* __restrict__ kv_layer, int S,
                                                      bf16* __restrict__ qout, int ldq) {
  pdl_trigger();
  pdl_wait();
  const int r = blockIdx.x;
  const int D = Hl * hd;
  const int vec = blockIdx.y * blockDim.x + threadIdx.x;      // vector index within the row's D
  if (vec * 8 >= D) return;
  const int e0 = vec * 8;
  const int h = e0 / hd, i0 = e0 - h * hd;
  const bf16* base = qkv + static_cast<size_t>(r) * ldq;
  float q[8], k[8], v[8];
  load16(base + e0, q);
  load16(base + D + e0, k);
  load16(base + 2 * D + e0, v);
  const int pos = row_pos[r];
  if (rot > 0 && i0 < rot) {
    const float fpos = static_cast<float>(pos);
    if (family == FL_FAMILY_GPTJ) {
      // interleaved pairs (2j, 2j+1) sit inside the vector: one sincos per pair
#pragma unroll
      for (int t = 0; t < 8; t += 2) {
        if (i0 + t >= rot) break;
        float sn, cs;
        rope_sincos(fpos, (i0 + t) >> 1, rot, &sn, &cs);
        const float q0 = q[t], q1 = q[t + 1], k0 = k[t], k1 = k[t + 1];
        q[t] = q0 * cs - q1 * sn;
        q[t + 1] = q1 * cs + q0 * sn;
        k[t] = k0 * cs - k1 * sn;
        k[t + 1] = k1 * cs + k0 * sn;
      }
    } else {
      // NeoX rotate-half: partner i +- rot/2 read element-wise from the row
      const int half = rot >> 1;
      float qo[8], ko[8];
#pragma unroll
      for (int t = 0; t < 8; ++t) {
        const int i = i0 + t;
        if (i >= rot) { qo[t] = q[t]; ko[t] = k[t]; continue; }
        const int j = i < half ? i : i - half;
        const int partner = i < half ? i + half : i - half;
        const float sign = i < half ? -1.f : 1.f;
        const float qp = __bfloat162float(base[h * hd + partner]);
        const float kp = __bfloat162float(base[D + h * hd + partner]);
        float sn, cs;
        rope_sincos(fpos, j, rot, &sn, &cs);
        qo[t] = q[t] * cs + sign * qp * sn;
        ko[t] = k[t] * cs + sign * kp * sn;
      }
#pragma unroll
      for (int t = 0; t < 8; ++t) { q[t] = qo[t]; k[t] = ko[t]; }
    }
  }
  store16(qout + static_cast<size_t>(r) * D + e0, q);
  const fl_row row = rows[r];
  if (row.kind != FL_ROW_ORPHAN) {
    const size_t kb = ((static_cast<size_t>(row.slot) * 2 + 0) * Hl + h) * S + pos;
    const size_t vb = ((static_cast<size_t>(row.slot) * 2 + 1) * Hl + h) * S + pos;
    store16(kv_layer + kb * hd + i0, k);
    store16(kv_layer + vb * hd + i0, v);
  }
}

void launch_rope_append(const void* qkv, const fl_row* rows, const int32_t* row_pos, int M,
                        int Hl, int hd, int rot, int family, void* kv_layer, int C, int S,
                        void* qout, int dtype, cudaStream_t s, int ldq) {
  if (M <= 0) return;
  if (ldq <= 0) ldq = 3 * Hl * hd;
  dim3 grid(M, Hl);
  if (family == FL_FAMILY_GPT2) rot = 0;
  if (dtype == FL_DTYPE_BF16 && hd % 8 == 0) {
    const int vecs = Hl * hd / 8;
    const int bs = vecs < 256 ? (vecs + 31) / 32 * 32 : 256;
    launch_k(k_rope_append_v, dim3(M, (vecs + bs - 1) / bs), dim3(bs), 0, s, 1, (const bf16*)qkv, rows, row_pos,
             Hl, hd, rot, family, (bf16*)kv_layer, S, (bf16*)qout, ldq);
    return;
  }
  if (dtype == FL_DTYPE_BF16)
    launch_k(k_rope_append<bf16>, dim3(grid), dim3(hd), 0, s, 1, (const bf16*)qkv, rows, row_pos, Hl, hd, rot, family,
                                            (bf16*)kv_layer, C, S, (bf16*)qout, ldq);
  else
    launch_k(k_rope_append<float>, dim3(grid), dim3(hd), 0, s, 1, (const float*)qkv, rows, row_pos, Hl, hd, rot,
                                             family, (float*)kv_layer, C, S, (float*)qout, ldq);
}

// ---------------------------------------------------------------- K8 greedy argmax
__global__ void __launch_bounds__(1024) k_argmax(const float* __restrict__ logits, int V, int ldl,
                                                 int index_base,
                                                 unsigned long long* __restrict__ keys) {
  pdl_trigger();
  pdl_wait();
  __shared__ unsigned long long red[32];
  const int r = blockIdx.x;
  const float* l = logits + static_cast<size_t>(r) * ldl;
  unsigned long long best = 0ull;
  for (int i = threadIdx.x; i < V; i += blockDim.x) {
    const unsigned long long k = argmax_key(l[i], index_base + i);
    best = k > best ? k : best;
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    const unsigned long long t = __shfl_xor_sync(0xffffffffu, best, o);
    best = t > best ? t : best;
  }
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = best;
  __syncthreads();
  if (threadIdx.x < 32) {
    best = threadIdx.x < (blockDim.x >> 5) ? red[threadIdx.x] : 0ull;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      const unsigned long long t = __shfl_xor_sync(0xffffffffu, best, o);
      best = t > best ? t : best;
    }
    if (threadIdx.x == 0) keys[r] = best;
  }
}

void launch_argmax(const float* logits, int M, int V, int ldl, int index_base,
                   unsigned long long* keys, cudaStream_t s) {
  if (M <= 0) return;
  launch_k(k_argmax, dim3(M), dim3(1024), 0, s, 1, logits, V, ldl, index_base, keys);
}

// ---------------------------------------------------------------- K9 state step
__global__ void k_apply_tokens(const unsigned long long* __restrict__ keys,
                               const fl_row* __restrict__ rows, const int32_t* __restrict__ row_pos,
                               int n_dec, int32_t* __restrict__ req_tok,
                               int32_t* __restrict__ req_pos, int32_t* __restrict__ req_ngen,
                               int32_t* __restrict__ tok_hist, int R, int max_new) {
  pdl_trigger();
  pdl_wait();
  const int r = blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= n_dec) return;
  const fl_row row = rows[r];
  if (row.kind != FL_ROW_DECODE) return;
  const int q = row.rid % R;
  const int tok = argmax_key_index(keys[r]);
  req_tok[q] = tok;
  req_pos[q] = row_pos[r] + 1;
  const int g = req_ngen[q];
  if (g < max_new) tok_hist[static_cast<size_t>(q) * max_new + g] = tok;
  req_ngen[q] = g + 1;
}

void launch_apply_tokens(const unsigned long long* keys, const fl_row* rows,
                         const int32_t* row_pos, int n_dec, int32_t* req_tok, int32_t* req_pos,
                         int32_t* req_ngen, int32_t* tok_hist, int R, int max_new, cudaStream_t s) {
  if (n_dec <= 0) return;
  launch_k(k_apply_tokens, dim3((n_dec + 127) / 128), dim3(128), 0, s, 1, keys, rows, row_pos, n_dec, req_tok, req_pos,
                                                     req_ngen, tok_hist, R, max_new);
}

}  // namespace fl

namespace fl {
// Weight re-layout for the tensor-core GEMM: W [N][K] row-major (rows K*2 bytes
// apart, so a 128-row x 64-column TMA box touches 128 DRAM pages) becomes
// [ceil(N/128)][K/64][128][64]: every box the GEMM loads is 16 KB contiguous
// (two consecutive K chunks of a tile are 32 KB contiguous).  Padding rows are
// zero.  One thread per 16-byte vector.
__global__ void k_tile_weight(const bf16* __restrict__ w, int N, int K, bf16* __restrict__ out) {
  const int kch = K / 64;
  const size_t n_vec = static_cast<size_t>((N + 127) / 128) * 128 * K / 8;
  for (size_t v = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x; v < n_vec;
       v += static_cast<size_t>(gridDim.x) * blockDim.x) {
    const size_t e = v * 8;                         // element index in the tiled layout
    const int c = static_cast<int>(e % 64);
    const size_t row = e / 64;                      // (tile * kch + kc) * 128 + r
    const int r = static_cast<int>(row % 128);
    const size_t tk = row / 128;
    const int kc = static_cast<int>(tk % kch);
    const size_t tile = tk / kch;
    const size_t n = tile * 128 + r;
    uint4 val = make_uint4(0u, 0u, 0u, 0u);
    if (n < static_cast<size_t>(N)) val = *reinterpret_cast<const uint4*>(w + n * K + kc * 64 + c);
    *reinterpret_cast<uint4*>(out + e) = val;
  }
}

size_t tiled_weight_bytes(int N, int K) { return static_cast<size_t>((N + 127) / 128) * 128 * K * 2; }

int launch_tile_weight(const void* w, int N, int K, void* out, cudaStream_t s) {
  if (N <= 0 || K <= 0 || K % 64) return -1;
  k_tile_weight<<<1184, 256, 0, s>>>(static_cast<const bf16*>(w), N, K, static_cast<bf16*>(out));
  return cudaGetLastError() == cudaSuccess ? 0 : -1;
}
}  // namespace fl
