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
#ifndef ATT_CW
#define ATT_CW 4   // consumer warps per CTA (A/B builds: 8 = one CTA per SM)
#endif
// K/V ring bytes per CTA.  The consumers are latency-bound (ncu at C4, hd 96:
// 2.4 active / 0.56 eligible warps per scheduler, issue slots 44 % busy), so
// smaller rings that let more CTAs share an SM win: 44 KB below head_dim 128
// (4 CTAs per SM, register-limited; C4 48 rows 10.54 -> 10.03 ms per
// iteration, C2 16 rows 463 -> 455 us), 64 KB from 128 (3 CTAs per SM with
// 8 KB K tiles; C3 128 rows 5932 -> 5896 us, 224 rows ~ -1 %)
#ifndef ATT_RING_SMALL
#define ATT_RING_SMALL 45056
#endif
#ifndef ATT_RING_LARGE
#define ATT_RING_LARGE 65536
#endif
#ifndef ATT_TILE_BYTES
#define ATT_TILE_BYTES 0   // 0: per head_dim (AttnCfg::TKB); A/B builds override
#endif

__device__ unsigned long long* g_att_dbg = nullptr;   // fl_attention_debug
void attn_set_debug(unsigned long long* p) { cudaMemcpyToSymbol(g_att_dbg, &p, sizeof(p)); }
FL_DEV unsigned long long gtime() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

int attn_max_splits(int S) { return (S + ATT_CHUNK - 1) / ATT_CHUNK; }

template <int X> struct NextPow2 {
  static constexpr int v = X <= 1 ? 1 : X <= 2 ? 2 : X <= 4 ? 4 : X <= 8 ? 8 : X <= 16 ? 16 : 32;
};

// split rows' contexts (flash-decoding + combine) only below one item per
// SM: between 148 and 296 (row, head) items the combine pass costs more than
// the idle half of the second CTA slots (C3 at 16 rows 2836 -> 2772 us per
// iteration; 64 loses at C2 8 rows: tools/prof_step.py)
#ifndef ATT_SPLIT_BELOW
#define ATT_SPLIT_BELOW 148
#endif
#ifndef ATT_SPLIT_TARGET
#define ATT_SPLIT_TARGET (2 * 148)
#endif
int attn_keys_per_split(int row_heads, int S) {
  const int full = attn_max_splits(S);
  int splits = 1;
  if (row_heads < ATT_SPLIT_BELOW) splits = (ATT_SPLIT_TARGET + row_heads - 1) / row_heads;
  if (splits > full) splits = full;
  const int keys = (S + splits - 1) / splits;
  return (keys + ATT_CHUNK - 1) / ATT_CHUNK * ATT_CHUNK;
}

// ---------------------------------------------------------------------------
// Persistent, TMA-staged decode attention.
//
// Work items are (row, head, split) triples; a grid of ~2 CTAs per SM walks
// them round-robin.  Warp CW (the producer) streams each item's K and V rows
// tile by tile with 1-D bulk copies (cp.async.bulk ... mbarrier::complete_tx)
// into a STAGES-deep shared-memory ring and runs ahead across item
// boundaries, so HBM sees a continuous stream.  CW consumer warps read the
// tiles from shared memory with 16-byte vector loads: a lane group of G
// lanes owns one key at a time (dot product + shuffle reduction), keeps its
// own online-softmax state (m, l, acc) and the groups are merged through
// shared memory at the end of the item -- no per-tile block barriers.
template <typename T, int HD>
struct AttnCfg {
  static constexpr int VEC = 16 / sizeof(T);             // elements per 16-byte vector
  static constexpr int NV = HD / VEC;                     // vectors per K/V row
  // 8 lanes per key: 3-level shuffle reductions and 4 independent keys per
  // warp-step; a warp-wide 16-byte load then spans 4 K rows (4 wavefronts,
  // the minimum for 512 bytes) so the layout costs no extra bank conflicts
  // (hd 96, bf16: 12 vectors -> 4 lanes x 3 instead of 8 lanes x 2 with a
  // quarter of the lanes idle, and 2 shuffle levels for 8 keys per warp-step)
  static constexpr int G0 = NextPow2<NV>::v < 8 ? NextPow2<NV>::v : 8;
  static constexpr int G = (NV % G0 == 0 || NV % 4 != 0) ? G0 : 4;   // lanes per key
  static constexpr int PER = (NV + G - 1) / G;            // vectors per lane
  static constexpr int KPW = 32 / G;                      // keys per warp-step
  static constexpr int CW = ATT_CW;                       // consumer warps
  static constexpr int THREADS = (CW + 1) * 32;
  static constexpr int ROW = HD * sizeof(T);              // bytes per key row
  // K bytes per tile: 8 KB (finer tiles keep more of the ring in flight:
  // hd 96 5.07 -> 5.50 TB/s at 2 CTAs per SM, tools/attn_bench.py; at head_dim
  // 256 16 KB tiles won at 2 CTAs per SM, 8 KB wins with 3 and a 64 KB ring)
  static constexpr int TKB = ATT_TILE_BYTES ? ATT_TILE_BYTES : 8192;
  static constexpr int TK = (TKB / ROW) / (CW * KPW) * (CW * KPW) > 0 ? (TKB / ROW) / (CW * KPW) * (CW * KPW)
                                                                      : CW * KPW;   // keys per tile
  // ring budget per CTA (the launcher sizes the grid by the co-resident CTAs per SM)
  static constexpr int RING = ATT_CW >= 8 ? 6 * 32768 : HD < 128 ? ATT_RING_SMALL : ATT_RING_LARGE;
  static constexpr int STAGES = (RING / 2) / (TK * ROW) < 2 ? 2 : (RING / 2) / (TK * ROW);
  static constexpr int STAGE_BYTES = 2 * TK * ROW;        // K tile + V tile
  static constexpr int SMEM = STAGES * STAGE_BYTES;
  // co-resident CTAs per SM the ring sizes are chosen for (register cap)
  static constexpr int MINB = ATT_CW >= 8 ? 1 : HD < 128 ? 4 : 3;
  // two keys per lane group and warp-step (one softmax rescale for both):
  // only where a tile holds >= 2 steps per warp without costing registers --
  // head_dim 64 (C2 16 rows 453.5 -> 446.7 us per iteration); at 96 / 256 it
  // needs 16 KB tiles and spills or loses a CTA per SM (C4 +5 %, C3 +1.3 %)
  static constexpr bool PAIR = HD <= 64;
};

FL_DEV uint32_t smem_addr(const void* p) { return static_cast<uint32_t>(__cvta_generic_to_shared(p)); }

FL_DEV void mbar_init_(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_addr(bar)), "r"(count));
}
FL_DEV void mbar_expect_tx_(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_addr(bar)),
               "r"(bytes) : "memory");
}
FL_DEV void mbar_arrive_(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_addr(bar)) : "memory");
}
FL_DEV void mbar_wait_(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred done;\n"
      "AWAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 done, [%0], %1;\n\t"
      "@!done bra AWAIT_%=;\n\t}" ::"r"(smem_addr(bar)), "r"(parity) : "memory");
}
FL_DEV void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          smem_addr(dst)),
      "l"(reinterpret_cast<uint64_t>(src)), "r"(bytes), "r"(smem_addr(bar))
      : "memory");
}

template <typename T>
FL_DEV void widen16(const uint4& raw, float* out) {
  if constexpr (sizeof(T) == 4) {
    out[0] = __uint_as_float(raw.x); out[1] = __uint_as_float(raw.y);
    out[2] = __uint_as_float(raw.z); out[3] = __uint_as_float(raw.w);
  } else {
    const __nv_bfloat162* h = reinterpret_cast<const __nv_bfloat162*>(&raw);
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      float2 f = __bfloat1622float2(h[j]);
      out[2 * j] = f.x; out[2 * j + 1] = f.y;
    }
  }
}

template <typename T, int HD>
__global__ void __launch_bounds__(AttnCfg<T, HD>::THREADS, AttnCfg<T, HD>::MINB) k_attn_tma(
    const T* __restrict__ q, const fl_row* __restrict__ rows, const int32_t* __restrict__ row_ctx,
    int M, int Hl, const T* __restrict__ kv_layer, int S, T* __restrict__ out,
    float* __restrict__ ws_o, float* __restrict__ ws_ml, int max_splits, int keys_per_split,
    int splits, const int4* __restrict__ meta, int ldo, unsigned* __restrict__ ctr,
    unsigned* __restrict__ next_ctr, unsigned* __restrict__ pre, int pre_mode) {
  using Cfg = AttnCfg<T, HD>;
  constexpr int VEC = Cfg::VEC, NV = Cfg::NV, G = Cfg::G, PER = Cfg::PER, KPW = Cfg::KPW;
  constexpr int CW = Cfg::CW, TK = Cfg::TK, STAGES = Cfg::STAGES, NP = CW;
  extern __shared__ __align__(128) uint8_t smem[];
  __shared__ __align__(8) uint64_t full[STAGES];
  __shared__ __align__(8) uint64_t empty[STAGES];
  __shared__ float s_m[NP], s_l[NP];
  __shared__ __align__(16) float s_acc[NP][HD];
  // items are handed out dynamically (one atomic per item, in descending-cost
  // order): the producer claims the next item and passes it to the consumers
  // through a small smem queue -- a CTA that runs fast takes more items
  constexpr int QD = 4;
  __shared__ int q_item[QD][4];                       // item, row, head, context
  __shared__ __align__(16) T q_s[QD][HD];             // the item's query (bulk copy)
  __shared__ __align__(8) uint64_t q_full[QD];
  __shared__ __align__(8) uint64_t q_empty[QD];

  pdl_trigger();    // the successor launches now; its griddepcontrol.wait waits for this grid
  unsigned long long* const dbg = g_att_dbg ? g_att_dbg + 64 * blockIdx.x : nullptr;
  if (dbg && threadIdx.x == 0) dbg[0] = gtime();
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    for (int i = 0; i < STAGES; ++i) {
      mbar_init_(&full[i], 1);
      mbar_init_(&empty[i], CW);
    }
    for (int i = 0; i < QD; ++i) {
      mbar_init_(&q_full[i], 1);
      mbar_init_(&q_empty[i], CW);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();

  const int n_items = M * Hl * splits;
  const int D = Hl * HD;
  const size_t head_stride = static_cast<size_t>(S) * HD;

  if (warp == CW) {
    // ---------------- producer: one lane streams K/V tiles into the ring
    if (lane == 0) {
      int st = 0, qs = 0;
      uint32_t ph = 0, qph = 0;
      // Before the grid dependency resolves (pre_mode 1: a step-graph launch
      // that is not the step's last attention), stream up to a ring of this
      // CTA's first item from keys written by EARLIER graph launches: with
      // every kernel triggering its dependents at entry, only data from a
      // previous launch is safe here.  The item's (row, context, slot, old
      // keys) come from this step's k_row_order, which publishes
      // pre[1] = pre[0] + 1 after writing them (pre[0] is advanced by the
      // step's last attention launch, after its own dependency wait, so it is
      // stable for the whole step).  meta.w = keys [0, w) of the row that no
      // kernel of this step writes (decode: ctx - 1; prefill / orphan: 0).
      int n_pre = 0;
      if (pre_mode == 1 && meta && static_cast<int>(blockIdx.x) < n_items) {
        const unsigned want = __ldcg(pre) + 1u;
        for (;;) {
          unsigned f;
          asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(f) : "l"(pre + 1) : "memory");
          if (f == want) break;
          __nanosleep(32);
        }
        const int item = static_cast<int>(blockIdx.x);
        const int rh = item / splits;
        const int4 m = __ldcg(meta + rh / Hl);
        const int h = rh % Hl, ctx = m.y, safe = m.w;
        const size_t slot = static_cast<size_t>(m.z);
        const int k0 = (item % splits) * keys_per_split;
        const int k1 = min(ctx, k0 + keys_per_split);
        const T* Kb = kv_layer + ((slot * 2 + 0) * Hl + h) * head_stride;
        const T* Vb = kv_layer + ((slot * 2 + 1) * Hl + h) * head_stride;
        for (int t0 = k0; t0 < k1 && n_pre < STAGES; t0 += TK) {
          const int nk = min(TK, k1 - t0);
          if (t0 + nk > safe) break;
          uint8_t* buf = smem + st * Cfg::STAGE_BYTES;   // ring still empty: no slot wait
          mbar_expect_tx_(&full[st], 2u * nk * Cfg::ROW);
          bulk_g2s(buf, Kb + static_cast<size_t>(t0) * HD, nk * Cfg::ROW, &full[st]);
          bulk_g2s(buf + TK * Cfg::ROW, Vb + static_cast<size_t>(t0) * HD, nk * Cfg::ROW, &full[st]);
          if (++st == STAGES) { st = 0; ph ^= 1; }
          ++n_pre;
        }
      }
      pdl_wait();   // q, row_ctx, the counters and this step's K/V rows come from predecessors
      if (pre_mode == 2 && blockIdx.x == 0) pre[0] += 1u;   // the step's last attention: next step's epoch
      bool first = true;
      for (;;) {
        // CTA b starts with item b (the first round needs no atomic); later
        // items come from the counter, offset by the grid
        int item = first ? static_cast<int>(blockIdx.x) : static_cast<int>(gridDim.x + atomicAdd(ctr, 1u));
        first = false;
        if (item >= n_items) item = -1;
        int sp = 0, h = 0, r = 0, ctx = 0, k0 = 0;
        size_t slot = 0;
        if (item >= 0) {
          sp = item % splits;
          const int rh = item / splits;
          h = rh % Hl;
          if (meta) {                          // rank -> (row, context, slot): one 16-byte load
            const int4 m = meta[rh / Hl];
            r = m.x;
            ctx = m.y;
            slot = static_cast<size_t>(m.z);
          } else {
            r = rh / Hl;
            ctx = row_ctx[r];
            slot = rows[r].slot;
          }
          k0 = sp * keys_per_split;
          if (k0 >= ctx) continue;            // a split past this row's context: no work
        }
        // the consumers get the item's indices and its query through the
        // queue slot: no dependent global loads on their side per item
        mbar_wait_(&q_empty[qs], qph ^ 1);
        q_item[qs][0] = item;
        q_item[qs][1] = r;
        q_item[qs][2] = h;
        q_item[qs][3] = ctx;
        if (item >= 0) {
          mbar_expect_tx_(&q_full[qs], HD * sizeof(T));
          bulk_g2s(q_s[qs], q + static_cast<size_t>(r) * D + h * HD, HD * sizeof(T), &q_full[qs]);
        } else {
          mbar_arrive_(&q_full[qs]);
        }
        if (++qs == QD) { qs = 0; qph ^= 1; }
        if (item < 0) break;
        const int k1 = min(ctx, k0 + keys_per_split);
        const T* Kb = kv_layer + ((slot * 2 + 0) * Hl + h) * head_stride;
        const T* Vb = kv_layer + ((slot * 2 + 1) * Hl + h) * head_stride;
        for (int t0 = k0 + n_pre * TK; t0 < k1; t0 += TK) {
          const int nk = min(TK, k1 - t0);
          mbar_wait_(&empty[st], ph ^ 1);
          uint8_t* buf = smem + st * Cfg::STAGE_BYTES;
          mbar_expect_tx_(&full[st], 2u * nk * Cfg::ROW);
          bulk_g2s(buf, Kb + static_cast<size_t>(t0) * HD, nk * Cfg::ROW, &full[st]);
          bulk_g2s(buf + TK * Cfg::ROW, Vb + static_cast<size_t>(t0) * HD, nk * Cfg::ROW, &full[st]);
          if (++st == STAGES) { st = 0; ph ^= 1; }
        }
        n_pre = 0;
      }
    }
    return;
  }

  pdl_wait();
  // ---------------- consumers
  const int g = lane % G;           // lane within the key group
  const int kw = lane / G;          // key group within the warp

  const float scale = rsqrtf(static_cast<float>(HD));
  int n_done = 0;   // items finished (diagnostic stamps)
  int st = 0, qs = 0;
  uint32_t ph = 0, qph = 0;
  for (;;) {
    mbar_wait_(&q_full[qs], qph);
    if (dbg && threadIdx.x == 0) {
      if (n_done == 0) dbg[1] = gtime();
      if (n_done < 31) dbg[2 + 2 * n_done] = gtime();
    }
    const int item = q_item[qs][0];
    const int r = q_item[qs][1], h = q_item[qs][2], ctx = q_item[qs][3];
    float qv[PER][VEC], acc[PER][VEC];
    if (item >= 0) {
#pragma unroll
      for (int p = 0; p < PER; ++p) {
        const int vi = g + p * G;
#pragma unroll
        for (int j = 0; j < VEC; ++j) acc[p][j] = 0.f;
        if (vi < NV) {
          widen16<T>(*reinterpret_cast<const uint4*>(&q_s[qs][vi * VEC]), qv[p]);
#pragma unroll
          for (int j = 0; j < VEC; ++j) qv[p][j] *= scale;
        }
      }
    }
    __syncwarp();
    if (lane == 0) mbar_arrive_(&q_empty[qs]);
    if (++qs == QD) { qs = 0; qph ^= 1; }
    if (item < 0) break;
    const int sp = item % splits;
    const int k0 = sp * keys_per_split;
    const int k1 = min(ctx, k0 + keys_per_split);
    const int nsplit = (ctx + keys_per_split - 1) / keys_per_split;

    float m = -INFINITY, l = 0.f;

    for (int t0 = k0; t0 < k1; t0 += TK) {
      const int nk = min(TK, k1 - t0);
      mbar_wait_(&full[st], ph);
      const uint8_t* Ks = smem + st * Cfg::STAGE_BYTES;
      const uint8_t* Vs = Ks + TK * Cfg::ROW;
      if constexpr (Cfg::PAIR) {
      // two keys per lane group and step, one online-softmax rescale for
      // both: half the exp / acc-rescale chain per key
      for (int kb = warp * KPW; kb < nk; kb += 2 * CW * KPW) {
        const int ka = kb + kw, kc = ka + CW * KPW;
        const bool va = ka < nk, vc = kc < nk;     // vc implies va
        float2 a0 = make_float2(0.f, 0.f), a1 = a0, c0 = a0, c1 = a0;
#pragma unroll
        for (int p = 0; p < PER; ++p) {
          const int vi = g + p * G;
          if (vi < NV) {
            float kf[VEC], kg[VEC];
            if (va) widen16<T>(*reinterpret_cast<const uint4*>(Ks + ka * Cfg::ROW + vi * 16), kf);
            if (vc) widen16<T>(*reinterpret_cast<const uint4*>(Ks + kc * Cfg::ROW + vi * 16), kg);
#pragma unroll
            for (int j = 0; j < VEC; j += 2) {
              const float2 q2 = make_float2(qv[p][j], qv[p][j + 1]);
              if (va) {
                if ((j >> 1) & 1) a1 = __ffma2_rn(q2, make_float2(kf[j], kf[j + 1]), a1);
                else a0 = __ffma2_rn(q2, make_float2(kf[j], kf[j + 1]), a0);
              }
              if (vc) {
                if ((j >> 1) & 1) c1 = __ffma2_rn(q2, make_float2(kg[j], kg[j + 1]), c1);
                else c0 = __ffma2_rn(q2, make_float2(kg[j], kg[j + 1]), c0);
              }
            }
          }
        }
        float da = (a0.x + a0.y) + (a1.x + a1.y), dc = (c0.x + c0.y) + (c1.x + c1.y);
#pragma unroll
        for (int o = G / 2; o > 0; o >>= 1) {
          da += __shfl_xor_sync(0xffffffffu, da, o);
          dc += __shfl_xor_sync(0xffffffffu, dc, o);
        }
        if (va) {
          const float m_new = fmaxf(m, vc ? fmaxf(da, dc) : da);
          const float c = __expf(m - m_new);
          const float pa = __expf(da - m_new);
          const float pc = vc ? __expf(dc - m_new) : 0.f;
          l = l * c + (pa + pc);
          m = m_new;
          const float2 pa2 = make_float2(pa, pa), pc2 = make_float2(pc, pc), cc = make_float2(c, c);
#pragma unroll
          for (int p = 0; p < PER; ++p) {
            const int vi = g + p * G;
            if (vi < NV) {
              float vf[VEC], vg[VEC];
              widen16<T>(*reinterpret_cast<const uint4*>(Vs + ka * Cfg::ROW + vi * 16), vf);
              if (vc) widen16<T>(*reinterpret_cast<const uint4*>(Vs + kc * Cfg::ROW + vi * 16), vg);
#pragma unroll
              for (int j = 0; j < VEC; j += 2) {
                float2 a2 = __ffma2_rn(pa2, make_float2(vf[j], vf[j + 1]),
                                       __fmul2_rn(make_float2(acc[p][j], acc[p][j + 1]), cc));
                if (vc) a2 = __ffma2_rn(pc2, make_float2(vg[j], vg[j + 1]), a2);
                acc[p][j] = a2.x;
                acc[p][j + 1] = a2.y;
              }
            }
          }
        }
      }
      } else {
#pragma unroll 2
      for (int kb = warp * KPW; kb < nk; kb += CW * KPW) {
        const int k = kb + kw;
        const bool valid = k < nk;
        // four independent partial sums: the dot product is otherwise one
        // dependent FMA chain of PER*VEC links per key (latency-bound at the
        // ~2 consumer warps per scheduler the smem ring leaves room for)
        // (sm_100 packed FFMA2: two fp32 FMAs per instruction)
        float2 d2a = make_float2(0.f, 0.f), d2b = make_float2(0.f, 0.f);
        if (valid) {
#pragma unroll
          for (int p = 0; p < PER; ++p) {
            const int vi = g + p * G;
            if (vi < NV) {
              float kf[VEC];
              widen16<T>(*reinterpret_cast<const uint4*>(Ks + k * Cfg::ROW + vi * 16), kf);
#pragma unroll
              for (int j = 0; j < VEC; j += 2) {
                const float2 q2 = make_float2(qv[p][j], qv[p][j + 1]), k2 = make_float2(kf[j], kf[j + 1]);
                if ((j >> 1) & 1) d2b = __ffma2_rn(q2, k2, d2b);
                else d2a = __ffma2_rn(q2, k2, d2a);
              }
            }
          }
        }
        float dot = (d2a.x + d2a.y) + (d2b.x + d2b.y);
#pragma unroll
        for (int o = G / 2; o > 0; o >>= 1) dot += __shfl_xor_sync(0xffffffffu, dot, o);
        if (valid) {
          const float m_new = fmaxf(m, dot);
          const float c = __expf(m - m_new);
          const float pk = __expf(dot - m_new);
          l = l * c + pk;
          m = m_new;
#pragma unroll
          for (int p = 0; p < PER; ++p) {
            const int vi = g + p * G;
            if (vi < NV) {
              float vf[VEC];
              widen16<T>(*reinterpret_cast<const uint4*>(Vs + k * Cfg::ROW + vi * 16), vf);
              const float2 pk2 = make_float2(pk, pk), c2 = make_float2(c, c);
#pragma unroll
              for (int j = 0; j < VEC; j += 2) {
                const float2 a2 = __ffma2_rn(pk2, make_float2(vf[j], vf[j + 1]),
                                             __fmul2_rn(make_float2(acc[p][j], acc[p][j + 1]), c2));
                acc[p][j] = a2.x;
                acc[p][j + 1] = a2.y;
              }
            }
          }
        }
      }
      }
      __syncwarp();
      if (lane == 0) mbar_arrive_(&empty[st]);
      if (++st == STAGES) { st = 0; ph ^= 1; }
    }

    // ---- merge the KPW key groups of this warp (same dims per lane g) ...
#pragma unroll
    for (int o = G; o < 32; o <<= 1) {
      const float m_o = __shfl_xor_sync(0xffffffffu, m, o);
      const float l_o = __shfl_xor_sync(0xffffffffu, l, o);
      const float mx = fmaxf(m, m_o);
      const float c1 = mx == -INFINITY ? 0.f : __expf(m - mx);
      const float c2 = mx == -INFINITY ? 0.f : __expf(m_o - mx);
      l = l * c1 + l_o * c2;
#pragma unroll
      for (int p = 0; p < PER; ++p)
#pragma unroll
        for (int j = 0; j < VEC; ++j) {
          const float a_o = __shfl_xor_sync(0xffffffffu, acc[p][j], o);
          acc[p][j] = acc[p][j] * c1 + a_o * c2;
        }
      m = mx;
    }
    // ... then the CW warps through shared memory
    if (lane == 0) {
      s_m[warp] = m;
      s_l[warp] = l;
    }
    if (kw == 0) {
#pragma unroll
      for (int p = 0; p < PER; ++p) {
        const int vi = g + p * G;
        if (vi < NV) {
#pragma unroll
          for (int j = 0; j < VEC; ++j) s_acc[warp][vi * VEC + j] = acc[p][j];
        }
      }
    }
    asm volatile("bar.sync 1, %0;" ::"n"(CW * 32) : "memory");
    float Mx = -INFINITY;
#pragma unroll
    for (int i = 0; i < NP; ++i) Mx = fmaxf(Mx, s_m[i]);
    float L = 0.f;
#pragma unroll
    for (int i = 0; i < NP; ++i) L += s_m[i] == -INFINITY ? 0.f : s_l[i] * __expf(s_m[i] - Mx);
    for (int e = threadIdx.x; e < HD; e += CW * 32) {
      float o = 0.f;
#pragma unroll
      for (int i = 0; i < NP; ++i) o += s_m[i] == -INFINITY ? 0.f : s_acc[i][e] * __expf(s_m[i] - Mx);
      if (nsplit == 1) {
        out[static_cast<size_t>(r) * ldo + h * HD + e] = from_f<T>(o / L);
      } else {
        const size_t w = (static_cast<size_t>(r) * Hl + h) * max_splits + sp;
        ws_o[w * HD + e] = o;
        if (e == 0) {
          ws_ml[2 * w] = Mx;
          ws_ml[2 * w + 1] = L;
        }
      }
    }
    asm volatile("bar.sync 1, %0;" ::"n"(CW * 32) : "memory");   // merge buffers reused
    if (dbg && threadIdx.x == 0 && n_done < 31) dbg[3 + 2 * n_done] = gtime();
    ++n_done;
  }
  if (next_ctr) {
    // a chain of launches with one counter each: this launch arms the next
    // one's (that launch claims only after its grid dependency wait, i.e.
    // after this grid completed; the launch before this one, which used it,
    // completed before this grid's own wait returned) -- no exit atomic
    if (blockIdx.x == 0 && threadIdx.x == 0) *next_ctr = 0u;
    return;
  }
  // this CTA's producer claimed its last item before it sent the sentinel:
  // the last CTA to finish re-arms the item counter for the next launch
  if (threadIdx.x == 0 && atomicAdd(ctr + 1, 1u) == gridDim.x - 1) {
    ctr[0] = 0u;
    ctr[1] = 0u;
  }
}

template <typename T, int HD>
__global__ void k_attn_combine(const int32_t* __restrict__ row_ctx, int Hl,
                               const float* __restrict__ ws_o, const float* __restrict__ ws_ml,
                               int max_splits, int keys_per_split, T* __restrict__ out, int ldo) {
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
    out[static_cast<size_t>(r) * ldo + h * HD + e] = from_f<T>(o / L);
  }
}

template <typename T, int HD>
static int attn_launch(const void* q, const fl_row* rows, const int32_t* row_ctx, int M, int Hl,
                       const void* kv_layer, int S, int kps, void* out, float* ws_o, float* ws_ml,
                       const int4* meta, int ldo, cudaStream_t s, unsigned* ctr, unsigned* next_ctr,
                       unsigned* pre, int pre_mode) {
  using Cfg = AttnCfg<T, HD>;
  static int num_sms = 0, per_sm = 0;
  if (!num_sms) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&num_sms, cudaDevAttrMultiProcessorCount, dev);
    cudaFuncSetAttribute(k_attn_tma<T, HD>, cudaFuncAttributeMaxDynamicSharedMemorySize, Cfg::SMEM);
    // co-resident CTAs per SM (smem-limited: 2 with 96 KB rings)
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_attn_tma<T, HD>, Cfg::THREADS, Cfg::SMEM);
    if (per_sm < 1) per_sm = 1;
  }
  const int ms = attn_max_splits(S);           // workspace stride (CHUNK-sized splits)
  const int splits = (S + kps - 1) / kps;
  const int items = M * Hl * splits;
  const int grid = items < per_sm * num_sms ? items : per_sm * num_sms;
  launch_k(k_attn_tma<T, HD>, dim3(grid), dim3(Cfg::THREADS), Cfg::SMEM, s, 1, (const T*)q, rows,
           row_ctx, M, Hl, (const T*)kv_layer, S, (T*)out, ws_o, ws_ml, ms, kps, splits, meta, ldo, ctr,
           next_ctr, pre, pre ? pre_mode : 0);
  if (splits > 1) {
    launch_k(k_attn_combine<T, HD>, dim3(Hl, M), dim3(HD < 128 ? HD : 128), 0, s, 1, row_ctx, Hl,
             ws_o, ws_ml, ms, kps, (T*)out, ldo);
    return 2;
  }
  return 1;
}

// Row ranks by descending context (ties: lower row first) for the item
// order: one CTA; thread i counts the keys below its own (keys are unique:
// (~ctx, row)) -- M comparisons against smem broadcasts instead of a bitonic
// network's log2(M)^2 / 2 block barriers (9.4 -> ~1 us at 144 rows, and the
// step's first kernels wait on it).  meta[rank] = (row, ctx, slot, 0).
__global__ void __launch_bounds__(1024) k_row_order(const int32_t* __restrict__ row_ctx,
                                                   const fl_row* __restrict__ rows, int M,
                                                   int4* __restrict__ meta, unsigned* __restrict__ pre) {
  __shared__ unsigned long long key[1024];
  __shared__ int pf_slot[1024];   // slots that prefill rows of this step write
  __shared__ int n_pf;
  pdl_trigger();
  pdl_wait();
  if (threadIdx.x == 0) n_pf = 0;
  __syncthreads();
  for (int i = threadIdx.x; i < M; i += blockDim.x) {
    key[i] = (static_cast<unsigned long long>(0x7fffffffu - static_cast<uint32_t>(row_ctx[i])) << 32) | i;
    if (pre && rows[i].kind == FL_ROW_PREFILL) pf_slot[atomicAdd(&n_pf, 1)] = rows[i].slot;
  }
  __syncthreads();
  for (int i = threadIdx.x; i < M; i += blockDim.x) {
    const unsigned long long k = key[i];
    int rank = 0;
    for (int j = 0; j < M; ++j) rank += key[j] < k;
    const int ctx = row_ctx[i];
    const fl_row ri = rows[i];
    // keys no kernel of this step writes (attention may stream them before its
    // grid dependency wait): a decode row appends key ctx - 1 this step, and
    // a request admitted this step has its prompt written by prefill rows
    int old = ri.kind == FL_ROW_DECODE ? ctx - 1 : 0;
    for (int j = 0; j < n_pf && old > 0; ++j)
      if (pf_slot[j] == ri.slot) old = 0;
    meta[rank] = make_int4(i, ctx, ri.slot, old > 0 ? old : 0);
  }
  if (pre) {
    __syncthreads();
    if (threadIdx.x == 0) {
      __threadfence();
      const unsigned v = __ldcg(pre) + 1u;
      asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(pre + 1), "r"(v) : "memory");
    }
  }
}

void launch_row_order(const int32_t* row_ctx, const fl_row* rows, int M, int4* meta, cudaStream_t s,
                      unsigned* pre) {
  if (M <= 0 || M > 1024) return;
  launch_k(k_row_order, dim3(1), dim3((M + 31) / 32 * 32), 0, s, 1, row_ctx, rows, M, meta, pre);
}

int launch_attention(const void* q, const fl_row* rows, const int32_t* row_ctx, int M, int Hl,
                     int hd, const void* kv_layer, int C, int S, int kps, void* out, float* ws_o,
                     float* ws_ml, int dtype, cudaStream_t s, const int4* meta, int ldo, unsigned* ctr,
                     unsigned* next_ctr, unsigned* pre, int pre_mode) {
  if (ldo <= 0) ldo = Hl * hd;
  if (M <= 0) return 0;
#define FL_ATT(HDV)                                                                          \
  case HDV:                                                                                  \
    return dtype == FL_DTYPE_BF16                                                            \
               ? attn_launch<bf16, HDV>(q, rows, row_ctx, M, Hl, kv_layer, S, kps, out, ws_o, \
                                        ws_ml, meta, ldo, s, ctr, next_ctr, pre, pre_mode)                  \
               : attn_launch<float, HDV>(q, rows, row_ctx, M, Hl, kv_layer, S, kps, out,      \
                                         ws_o, ws_ml, meta, ldo, s, ctr, next_ctr, pre, pre_mode);
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
