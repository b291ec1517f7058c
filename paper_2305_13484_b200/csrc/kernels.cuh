// Launchers for the fused decode step kernels (host side, internal).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include "../../include/flover_b200.h"

namespace fl {

enum Epilogue {
  EPI_STORE = 0,      // out(T)   = acc + bias
  EPI_GELU = 1,       // out(T)   = gelu(acc + bias)
  EPI_ACC_F32 = 2,    // out(f32) += acc + bias      (residual update)
  EPI_STORE_F32 = 3,  // out(f32) = acc + bias       (partial sums, logits)
  EPI_ARGMAX = 4      // keys[m] = max(keys[m], key(acc + bias, n))  (fused greedy argmax)
};

struct GemmArgs {
  const void* x;      // [M, K] activations, row stride ldx (elements)
  const void* w;      // [N, K] weights, row stride K
  const void* bias;   // [N] or null (same dtype as w)
  void* out;          // [M, N] row stride ldo
  int M, N, K, ldx, ldo;
  int epi;
  int dtype;          // FL_DTYPE_*
  int mcap;           // rows allocated behind x (>= M); fixes the TMA map per buffer
  unsigned long long* keys = nullptr;   // EPI_ARGMAX: per-row packed (logit, index) keys
  int index_base = 0;                   // EPI_ARGMAX: global index of weight row 0
  int w_tiled = 0;                      // w in the fl_tile_weight layout
  // two GEMMs over one weight stream [W1; W2] (EPI_GELU only, tcgen05 path):
  // weight rows n < nsplit read x and store plainly to out column n; rows
  // n >= nsplit read x2 (null: x) and get GELU, stored to column n + ogap.
  // nsplit is a multiple of 256 (whole pair tiles on either side).
  const void* x2 = nullptr;
  int nsplit = 0, ogap = 0;
  // no cross-CTA waits (whole tiles, one per CTA pair, grid not co-resident):
  // for launches that may share the GPU with another stream's GEMMs
  int indep = 0;
};

// SIMT FFMA GEMM (fp32 path and the reference path for the tensor-core GEMM).
void gemm_simt(const GemmArgs& a, cudaStream_t s);

// Resolve rows (token / position / context per row) and gather embeddings.
// Also zeroes keys[0, n_dec) for this step's greedy argmax.
void launch_embed(const fl_row* rows, int n_rows, int n_dec, const int32_t* req_tok,
                  const int32_t* req_pos, int32_t* req_ngen, int R, const void* wte,
                  const void* wpe, int d, int dtype, float* x, int32_t* row_tok, int32_t* row_pos,
                  int32_t* row_ctx, unsigned long long* keys, cudaStream_t s);

// out(T)[M, d] = LN(x[M, d]) * g + b
void launch_layernorm(const float* x, const void* g, const void* b, void* out, int M, int d,
                      float eps, int dtype, cudaStream_t s);
// two LayerNorms of the same rows in one launch (gridDim.y = 2)
void launch_layernorm2(const float* x, const void* g, const void* b, void* out, const void* g2,
                       const void* b2, void* out2, int M, int d, float eps, int dtype, cudaStream_t s);

// x += y + b1 (+ b2)   (after a tensor-parallel all-reduce of y)
void launch_add_partial(float* x, const float* y, const void* b1, const void* b2, int M, int d,
                        int dtype, cudaStream_t s);

// rotary on q/k, q -> qout [M, Hl*hd]; k/v -> KV pool of this layer at (slot, pos).
// qkv rows are ldq elements apart (0: 3 * Hl * hd).
void launch_rope_append(const void* qkv, const fl_row* rows, const int32_t* row_pos, int M,
                        int Hl, int hd, int rot, int family, void* kv_layer, int C, int S,
                        void* qout, int dtype, cudaStream_t s, int ldq = 0);

// split-K masked decode attention over each row's own context.
int attn_max_splits(int S);
// keys per split: one split per (row, head) when rows*heads fill the GPU.
int attn_keys_per_split(int row_heads, int S);
// returns the number of kernels launched (1 or 2)
// ctr: two zero-initialised device counters (item claims, finished CTAs);
// the kernel re-arms them, so one pair per stream of launches suffices.
// next_ctr (a chain of launches, one counter each, >= 2 in the cycle): the
// launch zeroes the next launch's claim counter instead of re-arming its own
// at exit
int launch_attention(const void* q, const fl_row* rows, const int32_t* row_ctx, int M, int Hl,
                     int hd, const void* kv_layer, int C, int S, int keys_per_split, void* out,
                     float* ws_o, float* ws_ml, int dtype, cudaStream_t s, const int4* meta,
                     int ldo, unsigned* ctr, unsigned* next_ctr = nullptr, unsigned* pre = nullptr,
                     int pre_mode = 0);
// meta[i] = (row, context, KV slot, keys not written this step) of rank i by
// descending context (attention's item order; M <= 1024).  pre (step graphs
// only): two words {epoch, published}; the kernel sets published = epoch + 1
// after meta, so attention launches (pre_mode 1) may stream their first
// item's older keys before their grid dependency wait; the step's last
// attention launch (pre_mode 2) advances the epoch after its wait.
void launch_row_order(const int32_t* row_ctx, const fl_row* rows, int M, int4* meta, cudaStream_t s,
                      unsigned* pre = nullptr);

// per-row (max logit, lowest index) as a packed 64-bit key
void launch_argmax(const float* logits, int M, int V, int ldl, int index_base,
                   unsigned long long* keys, cudaStream_t s);

// greedy token -> per-request state and token history
void launch_apply_tokens(const unsigned long long* keys, const fl_row* rows,
                         const int32_t* row_pos, int n_dec, int32_t* req_tok, int32_t* req_pos,
                         int32_t* req_ngen, int32_t* tok_hist, int R, int max_new, cudaStream_t s);

// K10: move live KV prefixes between physical slots
void launch_kv_copy(const int32_t* moves, int n_moves, const void* src_kv, int src_C, int src_S, void* dst_kv,
                    int dst_C, int dst_S, int L, int Hl, int hd, int dtype, cudaStream_t s);
void launch_shuffle_planned(const int32_t* plan, const int32_t* ctx_of, int lo, int max_moves, void* kv, int L,
                            int C, int Hl, int S, int hd, int dtype, cudaStream_t s);
void launch_shuffle(const int32_t* moves, int n_moves, void* kv, int L, int C, int Hl, int S,
                    int hd, int dtype, cudaStream_t s);

}  // namespace fl
