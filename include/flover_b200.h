/*
 * flover_b200.h -- C-ABI of the B200 fused decode loop (Flover, arXiv 2305.13484).
 *
 * The reference (fusionsim, /root/reference/pkg/src/fusionsim) is a pure-Python
 * simulator with no FFI; its fused loop *models* each device action.  Each entry
 * point below is the device realisation of one modelled action and sits directly
 * under the Python call that used to model it (see INTEGRATION.md for the
 * ctypes binding the drop-in engine uses):
 *
 *   fl_create / fl_destroy    -- FusionStream construction / teardown
 *                                (engine.py:48-85); device state is caller-owned.
 *   fl_step                   -- one atomic iteration FusionStream.step_iteration
 *                                (engine.py:128-160): every fused request gains one
 *                                token; the reference only charges
 *                                cost.iteration_time (cost.py:89-109) for it.
 *                                Newly fused requests (try_fuse_pending,
 *                                engine.py:97-124; preprocess engine.py:24-42) enter
 *                                as PREFILL rows of the same launch sequence.
 *   fl_shuffle                -- apply_shuffle (buffer.py:261-278) on the KV pool:
 *                                the move list of plan_shuffle (buffer.py:226-258);
 *                                the reference only charges shuffle_time
 *                                (cost.py:119-123).
 *   fl_comm_*                 -- the tensor-parallel communicator the reference
 *                                models as TPConfig + comm_time (cost.py:26-33,73-86).
 *
 * Conventions: every pointer to device memory is owned by the caller (PyTorch);
 * the library never allocates or frees caller memory.  All calls are stream-
 * ordered and non-blocking unless stated.  Return 0 on success, a negative
 * FL_E* code on failure (fl_last_error() has the message); no C++ exception
 * crosses the ABI.  One host thread per handle.
 */
#ifndef FLOVER_B200_H
#define FLOVER_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define FL_ABI_VERSION 1

enum fl_status {
  FL_OK = 0,
  FL_EINVAL = -1,     /* -> errors.InvalidParam      */
  FL_ECAPACITY = -2,  /* -> errors.CapacityExceeded  */
  FL_ESTALE = -3,     /* -> errors.StalePlan         */
  FL_ECUDA = -4,      /* -> errors.DeviceError       */
  FL_ENCCL = -5       /* -> errors.DeviceError       */
};

enum fl_family {
  FL_FAMILY_GPT2 = 0, /* sequential pre-LN blocks, learned positions, GELU MLP   */
  FL_FAMILY_GPTJ = 1, /* parallel residual, 1 LN, interleaved rotary (rotary_dim) */
  FL_FAMILY_NEOX = 2  /* parallel residual, 2 LNs, rotate-half rotary             */
};

enum fl_dtype { FL_DTYPE_F32 = 0, FL_DTYPE_BF16 = 1 };

enum fl_row_kind {
  FL_ROW_DECODE = 0,  /* fused request: input token/pos from per-request state (or explicit) */
  FL_ROW_PREFILL = 1, /* prompt token of a request fused at this boundary (no LM head)       */
  FL_ROW_ORPHAN = 2   /* evicted slot still inside the live window (fusion_noshuffle):       */
                      /* computed over stale KV, output discarded             */
};

/* Per-layer weight slots of fl_model_desc.layers (row-major [out, in] matrices). */
enum fl_layer_tensor {
  FL_W_LN1_G = 0, FL_W_LN1_B, FL_W_LN2_G, FL_W_LN2_B,
  FL_W_QKV,    /* [3 * Hl * hd, d]  rows: q heads, k heads, v heads (this rank) */
  FL_W_QKV_B,  /* [3 * Hl * hd] or NULL                                         */
  FL_W_O,      /* [d, Hl * hd]  row-parallel slice                              */
  FL_W_O_B,    /* [d] or NULL (added once, after the all-reduce)                */
  FL_W_FC,     /* [Fl, d]                                                       */
  FL_W_FC_B,   /* [Fl]                                                          */
  FL_W_PROJ,   /* [d, Fl]                                                       */
  FL_W_PROJ_B, /* [d]                                                           */
  FL_W_LAYER_COUNT
};

typedef struct fl_model_desc {
  int32_t family, dtype;
  int32_t n_layer, d_model, n_head, head_dim, d_ff, vocab, max_pos, rotary_dim;
  float ln_eps;
  int32_t tp_rank, tp_size;    /* heads, FFN columns and vocab are split tp_size ways */
  const void* wte;             /* [vocab, d] token embedding (replicated)             */
  const void* wpe;             /* [max_pos, d] learned positions or NULL              */
  const void* lnf_g;
  const void* lnf_b;
  const void* w_lm;            /* [ceil(vocab/tp), d] this rank's vocab slice          */
  const void* b_lm;            /* [ceil(vocab/tp)] or NULL                             */
  const void* const* layers;   /* host array [n_layer * FL_W_LAYER_COUNT]              */
} fl_model_desc;

typedef struct fl_pool_desc {
  int32_t pool_slots;       /* C: physical KV slots; logical slot s lives at s % C       */
  int32_t max_seq;          /* S: positions per slot (input_len + max_output - 1)        */
  int32_t max_rows;         /* rows per fused iteration (decode + orphan + prefill)      */
  int32_t state_slots;      /* R: per-request state ring, indexed rid % R                */
  int32_t max_new_tokens;   /* token history length per request                         */
  int32_t use_tensor_cores; /* 1: tcgen05 GEMMs (bf16 only), 2: same with weights tiled  */
                            /*    (fl_tile_weight); 0: SIMT FFMA GEMMs                   */
  void* kv;                 /* [L][C][2][Hl][S][hd] in the model dtype                   */
  int32_t* req_tok;         /* [R] next input token of a running request                 */
  int32_t* req_pos;         /* [R] position of that token                                */
  int32_t* req_ngen;        /* [R] tokens generated so far                               */
  int32_t* tok_hist;        /* [R][max_new_tokens] generated token ids                   */
  void* workspace;          /* fl_workspace_bytes() bytes, 256-B aligned                 */
  size_t workspace_bytes;
} fl_pool_desc;

/* One row of a fused iteration.  pos/tok < 0 on a DECODE row mean "read the
 * request's state" (the steady-state case: the host uploads nothing). */
typedef struct fl_row {
  int32_t slot;   /* physical KV slot                               */
  int32_t rid;    /* request id (state ring index = rid % R), -1 orphan */
  int32_t pos;    /* position of the input token, or -1              */
  int32_t tok;    /* input token id, or -1                            */
  int32_t kind;   /* fl_row_kind                                     */
  int32_t ctx;    /* ORPHAN only: stale context length to attend over */
} fl_row;

typedef struct fl_handle fl_handle;

int fl_abi_version(void);
const char* fl_last_error(void);

/* Bytes of scratch the caller must provide in fl_pool_desc.workspace. */
size_t fl_workspace_bytes(const fl_model_desc* model, const fl_pool_desc* pool);

int fl_create(const fl_model_desc* model, const fl_pool_desc* pool, fl_handle** out);
int fl_destroy(fl_handle* h);

/* Tensor parallelism: rank 0 calls fl_comm_unique_id, the id travels to every
 * rank (torch.distributed broadcast), then all ranks call fl_comm_init. */
int fl_comm_unique_id(void* out_128_bytes);
int fl_comm_init(fl_handle* h, const void* id_128_bytes, int rank, int world);

/* One fused iteration over rows[0..n_rows): rows [0, n_dec) are the live window
 * (DECODE / ORPHAN, window order), rows [n_dec, n_rows) are PREFILL rows.
 * rows is a HOST array, uploaded only when rows_changed != 0.  Greedy tokens of
 * DECODE rows update the per-request state and tok_hist on the device (no D2H).
 * logits_out (device fp32 [n_dec, vocab_local], may be NULL) receives the LM-head
 * output for parity checks. */
int fl_step(fl_handle* h, const fl_row* rows, int n_rows, int n_dec, int rows_changed,
            float* logits_out, void* cuda_stream);

/* K10: moves is a HOST array of n triples (src_slot, dst_slot, ctx_len) of
 * physical slots; copies the live KV prefix [0, ctx_len) of every
 * (layer, K/V, head) from src to dst in one launch.  Slots are disjoint. */
int fl_shuffle(fl_handle* h, const int32_t* moves, int n, void* cuda_stream);

/* Overlapped preprocessing (the paper's T_pp threads,
 * PAPER.md:231, which the reference models as an independent delay,
 * reference engine.py:6-8,24-42,69-83).  A second handle over the same
 * weights, created with a small STAGING pool (S = prompt length), runs the
 * prompts' PREFILL rows (n_dec = 0 fl_steps) on a side stream while the
 * serving handle's fused steps run on the main stream.
 *
 * fl_set_side_stream(h, 1): h's launches may share the GPU with another
 * handle's; its GEMMs then use decompositions without cross-CTA waits (one
 * whole tile per CTA pair), so neither stream's persistent grid can wait on
 * CTAs the other stream keeps from being resident.  Call before the first step.
 *
 * fl_step_import(h, staging kv, staging slots, staging S, moves, n): queue the
 * copy of prompt KV from staging slots into h's pool -- moves is a HOST array
 * of n triples (staging_slot, pool_slot, n_positions) -- to run at the start
 * of h's next fl_step, inside that step's timing bracket.  The caller orders
 * the staging writes before that step (an event from the side stream). */
int fl_set_side_stream(fl_handle* h, int on);
int fl_step_import(fl_handle* h, const void* src_kv, int src_slots, int src_seq, const int32_t* moves, int n);

/* Number of kernels fl_step / fl_shuffle launched since fl_create. */
int64_t fl_kernel_launches(const fl_handle* h);

/* Live kernel timing (CUDA events on the launch stream, bracketing each launch
 * group) for roofline reporting.  Classes: */
enum fl_prof_class {
  FL_PROF_ATTENTION = 0, /* K4 split + combine, one record per layer          */
  FL_PROF_GEMM = 1,      /* K3/K5/K6/K7/K8, one record per GEMM                */
  FL_PROF_SHUFFLE = 2,   /* K10, one record per fl_shuffle                     */
  FL_PROF_STEP = 3,      /* the whole fl_step                                  */
  FL_PROF_CLASSES = 4
};
/* Execution options: use_graphs (default 1) replays each (rows, window) shape
 * of fl_step as one CUDA graph; profile_every (default 8) samples one step in N
 * with event-bracketed launch groups while profiling is enabled; time_steps
 * brackets every fl_step / fl_shuffle with a pair of events (after any graph
 * capture work), read back by fl_last_duration_ms -- the engine's device clock. */
int fl_configure(fl_handle* h, int use_graphs, int profile_every, int time_steps);
/* Device time of the last fl_step or fl_shuffle (synchronises on it). */
int fl_last_duration_ms(fl_handle* h, float* ms);
int fl_profile(fl_handle* h, int enable);
/* Drains pending records (synchronises on them) and returns the totals since the
 * last fl_profile(h, 1): summed milliseconds, launch records, algorithmic bytes
 * and flops (GEMM: weights + activations in + out, 2*M*N*K; other classes 0). */
int fl_profile_read(fl_handle* h, int cls, double* total_ms, int64_t* records, double* bytes,
                    double* flops);

/* Diagnostic entry for kernel-level parity tests: one projection GEMM
 * out[M,N] (=|+=) X[M,K] . W[N,K]^T + bias through the same kernels fl_step
 * uses (use_tc: 1 tcgen05, 0 SIMT).  epi: 0 store(dtype) 1 gelu(dtype)
 * 2 accumulate(f32) 3 store(f32).  workspace: >= fl_gemm_workspace_bytes(). */
size_t fl_gemm_workspace_bytes(void);
/* Diagnostics: when non-NULL, every tensor-core GEMM CTA b writes 4 clocks to
 * dev_counters[4b..4b+3]: producer wait, producer total, MMA wait, MMA total. */
void fl_gemm_debug(unsigned long long* dev_counters);
/* Diagnostics: when non-NULL, every attention CTA b writes %globaltimer stamps to
 * dev_stamps[64b..64b+63]: [0] start, [1] after the grid dependency wait, then
 * per item i < 31: [2+2i] the consumers got the item, [3+2i] its output written. */
void fl_attention_debug(unsigned long long* dev_stamps);
/* Diagnostic entry: K4 alone.  q [M, Hl*hd]; rows (device) give the slot of each
 * row, row_ctx (device) its context length; kv_layer is one layer of the pool
 * [C][2][Hl][S][hd]; out [M, Hl*hd].  workspace >= fl_attention_workspace_bytes. */
size_t fl_attention_workspace_bytes(int M, int Hl, int hd, int S);
int fl_attention(const void* q, const fl_row* rows, const int32_t* row_ctx, int M, int Hl, int hd,
                 const void* kv_layer, int C, int S, void* out, void* workspace, int dtype,
                 void* cuda_stream);
int fl_gemm(const void* x, int ldx, const void* w, const void* bias, void* out, int ldo, int M,
            int N, int K, int epi, int dtype, int use_tc, void* workspace, void* cuda_stream);
/* Diagnostic entry, every epilogue: as fl_gemm, plus epi 4 = greedy argmax
 * (keys[m] = max(keys[m], packed(logit, index_base + n)); keys zeroed by the
 * caller, out unused) and the dual GEMM of fl_set_merged_in (nsplit > 0,
 * epi 1: weight rows >= nsplit read x2 and store GELU(.) at column n + ogap;
 * rows < nsplit read x and store plainly).  use_tc 2: W in fl_tile_weight
 * layout. */
int fl_gemm2(const void* x, const void* x2, int ldx, const void* w, const void* bias, void* out,
             int ldo, int M, int N, int K, int epi, int dtype, int use_tc, int nsplit, int ogap,
             unsigned long long* keys, int index_base, void* workspace, void* cuda_stream);
/* fl_gemm / fl_gemm2 re-arm the split-K flags of the caller's workspace on the
 * stream before every tensor-core call (default 1); timing loops over one
 * workspace may switch it off (the flags self-reset after each launch). */
void fl_gemm_set_rearm(int on);
/* Tuning studies only (tools/): key 0 = programmatic dependent launch (1 on,
 * 0 off) for every kernel launched afterwards; keys 1-4 override the GEMM's
 * work decomposition (max pairs, ring stages, K sub-chunks per unit, minimum
 * units per stream-K range); 5 span cap; 6-8 diagnostic switches (no loads /
 * no MMAs / no epilogue: garbage results); 9 = 1: fl_gemm_debug launches
 * alternate between two 64 K-entry halves of the buffer; -1 restores the
 * built-in choice. */
void fl_gemm_tune(int key, int value);

/* Parallel-residual families (gptj, neox): run the attention output projection
 * and the FFN down projection as ONE GEMM over K = Dl + Fl,
 *   x += [a | f] . [W_o | W_proj]^T + b_o + b_proj
 * (one reduction, and under tensor parallelism one all-reduce per layer instead
 * of two).  w_cat[l]: [d_model][Dl + Fl] in the layout the pool's
 * use_tensor_cores selects; b_cat[l]: b_o + b_proj or NULL (b_cat may be NULL).
 * Call after fl_create, before the first fl_step.  The per-layer W_O / W_PROJ
 * pointers are then unused. */
int fl_set_merged_out(fl_handle* h, const void* const* w_cat, const void* const* b_cat);

/* Parallel-residual families (gptj, neox), tensor-core pools: run the QKV
 * projection and the FFN up projection as ONE GEMM over the stacked weight
 * [W_qkv; W_fc] ([3Dl + Fl][d_model], the pool's layout), bias [b_qkv | b_fc]
 * (zeros where a model has none; b_in may be NULL).  Rows < 3Dl read LN1(x)
 * and store q|k|v; rows >= 3Dl read the MLP input (GPT-J: LN1(x), NeoX:
 * LN2(x)) and store GELU(FFN-up): one persistent launch balances both weight
 * streams over all SMs (QKV alone has fewer 256-row tiles than SM pairs).
 * Needs 3Dl % 256 == 0.  Windows of more than max_rows rows (< 0: the
 * default, 256) run QKV and FFN-up as two GEMMs over views of the stacked
 * weight (rows [0, 3Dl) and [3Dl, 3Dl + Fl)).  Call after fl_create, before
 * the first fl_step. */
int fl_set_merged_in(fl_handle* h, const void* const* w_in, const void* const* b_in, int max_rows);

/* Tensor-core weight layout: bytes of the tiled copy of a bf16 W [N][K]
 * (K % 64 == 0) and the stream-ordered re-layout into `out`.  A pool created
 * with use_tensor_cores = 2 expects every projection weight (w_qkv, w_o, w_fc,
 * w_proj of each layer, and w_lm) in this layout: [ceil(N/128)][K/64][128][64],
 * so each 128 x 64 tile the GEMM streams is 16 KB of contiguous memory. */
size_t fl_tiled_weight_bytes(int N, int K);
int fl_tile_weight(const void* w, int N, int K, void* out, void* cuda_stream);

/* Device-resident shuffle planner: Algorithm 1
 * (find_shuffled_memory_region, reference buffer.py:59-88) and plan_shuffle
 * (buffer.py:226-258) over one window of n <= 8192 slots starting at slot lo.
 * occ[n] (int32, nonzero = occupied) and size[n] (int64 bytes) are device
 * arrays.  Writes, stream-ordered, into device memory:
 *   out[0] = window offset (absolute slot), out[1] = window length (occupants),
 *   out[2] = n_moves, out[3 + 2r], out[4 + 2r] = (src, dst) slot of move r
 *   (ascending, as plan_shuffle pairs them);  *bytes = total_bytes_moved.
 * out must hold 3 + 2n ints.  Returns FL_EINVAL for n outside [0, 8192]. */
int fl_plan_shuffle(const int32_t* occ, const int64_t* size, int n, int lo, int32_t* out,
                    long long* bytes, void* cuda_stream);

/* A shuffle boundary planned and executed on the device: the
 * window's occupancy -- occ[n] (nonzero = occupied), size[n] (bytes, the
 * reference's tensor_size), ctx[n] (live KV positions of each occupant), HOST
 * arrays of window slots lo .. lo+n-1 -- is uploaded once; Algorithm 1 +
 * plan_shuffle run on the device (as fl_plan_shuffle) and K10 consumes the
 * device move list directly (physical slot = logical slot % pool_slots), so
 * the moves never pass through the host before the copy.  The plan (the
 * fl_plan_shuffle layout, 3 + 2n int32) and total_bytes_moved are copied,
 * stream-ordered, to plan_out / bytes_out (host, pinned; either may be NULL)
 * for the host's mirror of the layout.  With time_steps on, the device clock
 * covers planner + K10.  Replaces the host plan_shuffle / apply_shuffle pair
 * (reference buffer.py:226-278) on the device side. */
int fl_shuffle_planned(fl_handle* h, const int32_t* occ, const int64_t* size, const int32_t* ctx, int n, int lo,
                       int32_t* plan_out, long long* bytes_out, void* cuda_stream);

#ifdef __cplusplus
}
#endif
#endif /* FLOVER_B200_H */
