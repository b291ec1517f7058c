// K3/K5/K6/K7/K8 projections: persistent stream-K GEMM on 2-SM tcgen05 pairs.
//
// out[M,N] = X[M,K] . W[N,K]^T, swap-AB: a CTA pair (cluster of 2, one
// tcgen05.mma.cta_group::2 per K-step) owns a 256-row weight tile on the UMMA
// M side -- each CTA stages its own 128 weight rows and half of the window's
// token columns -- and the whole fused window (<= 512 tokens, MT sub-tiles of
// BN <= 256 columns) on the UMMA N side, accumulated in TMEM.
//
// Work decomposition (stream-K): the (token tile, weight tile, 64-wide K
// chunk) units of the GEMM are dealt out as equal contiguous ranges to one
// pair per two SMs, so every SM streams the same number of weight bytes no
// matter how N/256 divides 74 (QKV: 48 tiles, FFN-up: 64, attn-out: 16 ...).
// A range crosses weight tiles; the piece of a tile a pair owns is a
// "segment".  A tile split between pairs is finished by
//   - residual GEMMs (EPI_ACC_F32): every segment red.add.v4's its partial
//     into the fp32 residual (bias from the segment holding k = 0);
//   - all other epilogues: the segment holding k = 0 (always the LAST segment
//     of its pair's range, while the other pieces are the FIRST segments of
//     the following pairs' ranges) waits for the others' fp32 partials
//     (workspace slot per pair + release/acquire flag, self-resetting) and
//     runs the epilogue on the full sum.  Waits only point to higher pairs,
//     so they cannot cycle.
//
// Roles (256 threads per CTA):
//   warp 0   : TMA producer of the weight tiles (ahead of griddepcontrol.wait)
//   warps 6,7: TMA producers of the token sub-tiles
//   warp 1   : TMEM allocator; in the leader CTA lane 0 issues the MMAs
//   warps 2-5: epilogue (TMEM lanes 32*(warp%4)..+32), double-buffered TMEM
//              accumulators when the window fits 256 columns
// Reference: the modelled step is cost.py:89-109 (iteration_time); the GEMMs
// are the FC layers the paper shards across TP ranks.
#include <cudaTypedefs.h>

#include <cstdio>
#include <cstdlib>
#include <map>
#include <string>
#include <tuple>

#include "common.cuh"
#include "gemm_tc.cuh"

namespace fl {

namespace {

constexpr int SK_BM = 128;                 // weight rows per CTA (256 per pair)
constexpr int SK_BK = 64;                  // K per stage (one 128-byte swizzle row)
constexpr int SK_THREADS = 384;             // 12 warps: producers 0,6,7; MMA 1; epilogue 2-5, 8-11
constexpr int SK_A_BYTES = SK_BM * SK_BK * 2;
constexpr int SK_MAXST = 16;
constexpr int SK_MAXBUF = 4;               // TMEM accumulator buffers
constexpr int SK_RING_BUDGET = 200 * 1024;
constexpr int SK_STG_LD = 36;              // transpose row stride (floats): conflict-free

thread_local std::string g_sk_err;
// diagnostic overrides (fl_gemm_tune; -1 = the built-in choice): 1 max pairs,
// 2 ring stages, 3 K sub-chunks per unit, 4 min units per stream-K range,
// 5 tokens per token tile (span cap, <= 512)
int g_tune[10] = {-1, -1, -1, -1, -1, -1, -1, -1, -1, -1};
int g_l2_ahead = -1;                      // fl_gemm_tune key 8 (L2 prefetch depth / diagnostics)
unsigned long long* g_sk_dbg = nullptr;

FL_DEV uint32_t smem_u32(const void* p) { return static_cast<uint32_t>(__cvta_generic_to_shared(p)); }

FL_DEV void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}
FL_DEV void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
               : "memory");
}
FL_DEV bool mbar_try(uint64_t* bar, uint32_t parity) {
  uint32_t ok;
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
      "selp.u32 %0, 1, 0, p;\n\t}"
      : "=r"(ok)
      : "r"(smem_u32(bar)), "r"(parity)
      : "memory");
  return ok != 0;
}
// one waiting thread with back-off (keeps the MIO queue free for the others)
FL_DEV unsigned long long gtimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
FL_DEV void mbar_wait_sleep(uint64_t* bar, uint32_t parity) {
  while (!mbar_try(bar, parity)) __nanosleep(40);
}
FL_DEV void mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred done;\n"
      "WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 done, [%0], %1;\n\t"
      "@!done bra WAIT_%=;\n\t}" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}
// arrive on the barrier at the same smem offset in cluster CTA `rank`
FL_DEV void mbar_arrive_cluster(uint64_t* bar, uint32_t rank) {
  uint32_t remote;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(remote) : "r"(smem_u32(bar)), "r"(rank));
  // default semantics (release, CTA scope), as CUTLASS's ClusterBarrier::arrive:
  // the consumer's TMEM reads are ordered by tcgen05.wait::ld +
  // fence::before_thread_sync, and a cluster-scope release would also wait
  // for this thread's global stores
  asm volatile("mbarrier.arrive.shared::cluster.b64 _, [%0];" ::"r"(remote) : "memory");
}
// 2-SM load: lands in this CTA's smem, completes tx on the leader's barrier
FL_DEV void tma_load_pair(const CUtensorMap* map, uint64_t* bar, void* dst, int c0, int c1) {
  const uint32_t leader_bar = smem_u32(bar) & 0xFEFFFFFFu;
  asm volatile(
      "cp.async.bulk.tensor.2d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, "
      "{%3, %4}], [%2];" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(leader_bar), "r"(c0), "r"(c1)
      : "memory");
}
// 3-D variant: box {64, rows, kpb} of a [k/64][rows][64] view -> kpb stacked
// SW128 tiles in one request (a request costs its issuing thread a fixed
// ~250 cycles, so bigger boxes stream proportionally faster)
FL_DEV void tma_load_pair3(const CUtensorMap* map, uint64_t* bar, void* dst, int row, int kc) {
  const uint32_t leader_bar = smem_u32(bar) & 0xFEFFFFFFu;
  asm volatile(
      "cp.async.bulk.tensor.3d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, "
      "{%3, %4, %5}], [%2];" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(leader_bar), "r"(0), "r"(row), "r"(kc)
      : "memory");
}
FL_DEV void mma_pair(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc, uint32_t idesc, uint32_t acc) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem_d),
      "l"(adesc), "l"(bdesc), "r"(idesc), "r"(acc));
}
// Warp-uniform issue: the whole MMA warp runs the loop and one elected lane
// issues.  Descriptors computed in uniform control flow stay in uniform
// registers; issued from a lane-0 branch instead, every tcgen05.mma was
// wrapped in an ELECT loop with five R2UR.BROADCASTs (~165 clk per MMA
// against 82-94 clk back to back, tools/probes/mma2_probe.cu).
FL_DEV void mma_pair_elect(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc, uint32_t idesc, uint32_t acc) {
  asm volatile(
      "{\n\t.reg .pred p, e;\n\t"
      "elect.sync _|e, 0xffffffff;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "@e tcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem_d),
      "l"(adesc), "l"(bdesc), "r"(idesc), "r"(acc));
}
// One ring stage of a single token sub-tile with two 64-wide K chunks
// (kpb = 2, mt = 1, the common case): 8 MMAs in ONE asm block, descriptors
// stepped in PTX from three bases, so ptxas moves three values to uniform
// registers per stage instead of five per MMA.  The 16-deep K step is +32 B
// (+2 in the descriptor's 16-byte units), the second chunk of A is +16 KB.
FL_DEV void mma_stage2_elect(uint32_t tmem_d, uint64_t ad0, uint64_t bd0, uint64_t bd1, uint32_t idesc,
                             uint32_t acc_first) {
  asm volatile(
      "{\n\t.reg .pred e, p0, p1;\n\t.reg .b64 a, b;\n\t"
      "elect.sync _|e, 0xffffffff;\n\t"
      "setp.ne.b32 p0, %5, 0;\n\t"
      "setp.eq.b32 p1, %5, %5;\n\t"
      "@e tcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %4, p0;\n\t"
      "add.s64 a, %1, 2;\n\tadd.s64 b, %2, 2;\n\t"
      "@e tcgen05.mma.cta_group::2.kind::f16 [%0], a, b, %4, p1;\n\t"
      "add.s64 a, %1, 4;\n\tadd.s64 b, %2, 4;\n\t"
      "@e tcgen05.mma.cta_group::2.kind::f16 [%0], a, b, %4, p1;\n\t"
      "add.s64 a, %1, 6;\n\tadd.s64 b, %2, 6;\n\t"
      "@e tcgen05.mma.cta_group::2.kind::f16 [%0], a, b, %4, p1;\n\t"
      "add.s64 a, %1, 1024;\n\t"
      "@e tcgen05.mma.cta_group::2.kind::f16 [%0], a, %3, %4, p1;\n\t"
      "add.s64 a, %1, 1026;\n\tadd.s64 b, %3, 2;\n\t"
      "@e tcgen05.mma.cta_group::2.kind::f16 [%0], a, b, %4, p1;\n\t"
      "add.s64 a, %1, 1028;\n\tadd.s64 b, %3, 4;\n\t"
      "@e tcgen05.mma.cta_group::2.kind::f16 [%0], a, b, %4, p1;\n\t"
      "add.s64 a, %1, 1030;\n\tadd.s64 b, %3, 6;\n\t"
      "@e tcgen05.mma.cta_group::2.kind::f16 [%0], a, b, %4, p1;\n\t}" ::"r"(tmem_d),
      "l"(ad0), "l"(bd0), "l"(bd1), "r"(idesc), "r"(acc_first));
}
FL_DEV void commit_pair_elect(uint64_t* bar, uint16_t mask) {
  asm volatile(
      "{\n\t.reg .pred e;\n\t"
      "elect.sync _|e, 0xffffffff;\n\t"
      "@e tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;\n\t}"
      ::"r"(smem_u32(bar)), "h"(mask)
      : "memory");
}
// arrive on `bar` in both CTAs of the pair (mask = 3 << even rank of the pair)
FL_DEV void commit_pair(uint64_t* bar, uint16_t mask) {
  asm volatile(
      "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], "
      "%1;" ::"r"(smem_u32(bar)), "h"(mask)
      : "memory");
}
FL_DEV uint32_t cluster_ctarank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
FL_DEV void tc_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
FL_DEV void tc_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }
FL_DEV void cluster_sync_all() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
FL_DEV uint64_t desc_sw128(const void* tile) {
  const uint64_t addr = smem_u32(tile);
  uint64_t d = (addr >> 4) & 0x3FFFull;
  d |= 1ull << 16;
  d |= (1024ull >> 4) << 32;
  d |= 1ull << 46;
  d |= 2ull << 61;
  return d;
}
__host__ __device__ constexpr uint32_t idesc_bf16(int m, int n) {
  return (1u << 4) | (1u << 7) | (1u << 10) | (uint32_t(n >> 3) << 17) | (uint32_t(m >> 4) << 24);
}
FL_DEV void tmem_ld32(uint32_t taddr, uint32_t* r) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
      "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),
        "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]),
        "=r"(r[14]), "=r"(r[15]), "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]),
        "=r"(r[21]), "=r"(r[22]), "=r"(r[23]), "=r"(r[24]), "=r"(r[25]), "=r"(r[26]), "=r"(r[27]),
        "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
      : "r"(taddr));
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
}
FL_DEV void tmem_ld16(uint32_t taddr, uint32_t* r) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
        "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
      : "r"(taddr));
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
}
FL_DEV unsigned ld_acquire(const unsigned* p) {
  unsigned v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
FL_DEV void st_release(unsigned* p, unsigned v) {
  asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
FL_DEV void red_release_add(unsigned* p, unsigned v) {
  asm volatile("red.release.gpu.global.add.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
FL_DEV void epi_bar() { asm volatile("bar.sync 1, 256;" ::: "memory"); }   // the 8 epilogue warps

struct SkParams {
  int M, N, ldo, epi;
  int kch;          // K / 64
  int ntn;          // 256-row weight tiles
  int mt, bn;       // token sub-tiles per tile and their width (UMMA N)
  int span;         // tokens per token tile (mt * bn)
  int stages, ncols, nbuf;
  int units;        // ntm * ntn * kch
  int npairs;       // pairs in the grid = work ranges
  int dpw;          // whole tiles per pair in the data-parallel prefix (see pair_ranges)
  int nsk;          // pairs sharing the stream-K units after the prefix (<= npairs)
  const bf16* bias;
  void* out;
  unsigned long long* keys;
  int index_base;
  float* part;      // [npairs][2][span_max][128] fp32 partial slots
  unsigned* flags;  // [npairs][2]
  int slot_elems;   // floats per (pair, half) slot
  int vec;          // out rows 16-byte aligned: vector stores
  int csplit;       // >1: tile K split evenly over S pairs, spread reduction
  int red;          // EPI_ACC_F32: pieces of split tiles red.add into the residual (no fix-up)
  int slice;        // tokens per pair (mt * bn)
  int kpb;          // 64-wide K sub-chunks per unit/stage (2: one 3-D request per operand)
  int ntm;          // token tiles
  int w_tiled;      // weights in the fl_tile_weight layout [N/128][K/64][128][64]
  int kch64;        // K / 64
  int nsplit, ogap; // dual GEMM (GemmArgs::nsplit): rows >= nsplit read x2, GELU, column + ogap
  unsigned long long* dbg;   // diagnostics: per CTA [prod wait, prod total, mma wait, mma total]
  int dbg_skip_x;            // diagnostics (fl_gemm_tune 6): no activation loads
  int dbg_skip_mma;          // diagnostics (fl_gemm_tune 7): no MMAs (pipeline + epilogue only)
  int dbg_skip_epi;          // diagnostics (fl_gemm_tune 8 = -2): no epilogue (TMEM drained unread)
  int dbg_epi;               // diagnostics (key 8 = -10 - bits): 1 no GELU, 2 no output stores
  int l2_ahead;              // units of weights prefetched into L2 behind the ring fill
};

// dual GEMM: output column and activation of weight row n (identity / on
// for a single GEMM)
FL_DEV int ocol(const SkParams& P, int n) { return P.nsplit && n >= P.nsplit ? n + P.ogap : n; }
FL_DEV bool act_on(const SkParams& P, int n) { return !P.nsplit || n >= P.nsplit; }

// Work of pair q (unit index = tile * kch + K unit): a data-parallel prefix
// of dpw whole tiles [q*dpw, (q+1)*dpw), then an equal share of the units
// left after the npairs*dpw prefix tiles (stream-K) if q < nsk.  dpw = 0:
// pure stream-K (or the even split of csplit); no remainder: pure whole
// tiles.  Every pair streams the same number of weight bytes, all SMs busy
// whatever N/256 is.  nsk <= the remaining units, so no stream-K range is
// empty: every pair between a split tile's owner and its last piece holds a
// piece and publishes it (an empty one would leave the owner waiting).
struct Ranges {
  int lo[2], hi[2];
};
// Processing order: the stream-K share FIRST, then the whole tiles.  A split
// tile's pieces other than k = 0 are then the very first segments of the
// following pairs (published right away), and the k = 0 owner's fold-in and
// epilogue overlap the MMAs of its whole tiles instead of trailing the
// launch (an owner last in its range added ~8 us of exposed fix-up at 128
// tokens: tools/gemm_cta_dump.py).
FL_DEV Ranges pair_ranges(const SkParams& P, int q) {
  Ranges r;
  const int dpu = P.dpw * P.kch;
  r.lo[1] = q * dpu;
  r.hi[1] = r.lo[1] + dpu;
  const int base = dpu * P.npairs, ur = P.units - base;
  const int qs = q < P.nsk ? q : P.nsk;
  r.lo[0] = base + static_cast<int>((static_cast<long long>(qs) * ur) / P.nsk);
  r.hi[0] = q < P.nsk ? base + static_cast<int>((static_cast<long long>(q + 1) * ur) / P.nsk) : r.lo[0];
  return r;
}
// the pair whose stream-K range holds unit x (x past the whole-tile prefix)
FL_DEV int owner_of(int x, const SkParams& P) {
  const int base = P.dpw * P.kch * P.npairs, ur = P.units - base;
  return static_cast<int>(((static_cast<long long>(x - base) + 1) * P.nsk + ur - 1) / ur) - 1;
}
// one segment = the part of one tile inside one range
struct Seg {
  int t, klo, khi;
};
FL_DEV Seg seg_at(int u, int hi, int kch) {
  Seg g;
  g.t = u / kch;
  g.klo = u - g.t * kch;
  g.khi = min(kch, g.klo + (hi - u));
  return g;
}

enum { BLK_FINAL = 0, BLK_PUB = 2, BLK_RED = 3 };

// One 16-token block of one warp (lane = TMEM lane = weight row, r[j] = token
// cb + j) through the per-warp smem transpose: afterwards lane holds 4
// adjacent weight rows (c4) of tokens jb, jb + 4, jb + 8, jb + 12, so every
// access is 16 bytes.  PUB: fp32 partial to the pair's slot; RED: red.add
// into the fp32 residual.
template <int EPI, int MODE>
FL_DEV void block16(const SkParams& P, const uint32_t* r, float bv, float* ws_, int lane, int quarter, int nbase,
                    int m0, int cb, int ncol, float* pub) {
#pragma unroll
  for (int j = 0; j < 16; ++j) ws_[j * SK_STG_LD + lane] = __uint_as_float(r[j]) + bv;
  __syncwarp();
  const int c4 = (lane & 7) * 4, jb = lane >> 3;
  const int nn = nbase + quarter * 32 + c4;
  if (MODE == BLK_PUB) {
    float* dst = pub + static_cast<size_t>(cb) * SK_BM + quarter * 32 + c4;
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const int j = i * 4 + jb;
      if (j < ncol)
        *reinterpret_cast<float4*>(dst + j * SK_BM) = *reinterpret_cast<const float4*>(ws_ + j * SK_STG_LD + c4);
    }
  } else {
    float* dst = static_cast<float*>(P.out) + static_cast<size_t>(m0 + cb) * P.ldo + nn;
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const int j = i * 4 + jb;
      if (j < ncol) {
        const float4 v = *reinterpret_cast<const float4*>(ws_ + j * SK_STG_LD + c4);
        asm volatile("red.global.add.v4.f32 [%0], {%1, %2, %3, %4};" ::"l"(dst + static_cast<size_t>(j) * P.ldo),
                     "f"(v.x), "f"(v.y), "f"(v.z), "f"(v.w)
                     : "memory");
      }
    }
  }
  __syncwarp();
}

// Final epilogue of one 16-token block (whole tile, or the k = 0 owner of a
// split tile adding the later pieces' partials of pairs pair+1 .. plast).
template <int EPI>
FL_DEV void final16(const SkParams& P, const uint32_t* r, float bv, float* ws_, int lane, int quarter, int nbase,
                    int m0, int cb, int ncol, int pair, int plast, int xi) {
#pragma unroll
  for (int j = 0; j < 16; ++j) ws_[j * SK_STG_LD + lane] = __uint_as_float(r[j]) + bv;
  __syncwarp();
  const int c4 = (lane & 7) * 4, jb = lane >> 3;
  const int nn = nbase + quarter * 32 + c4;
  float4 w[4];
#pragma unroll
  for (int i = 0; i < 4; ++i) w[i] = *reinterpret_cast<const float4*>(ws_ + (i * 4 + jb) * SK_STG_LD + c4);
  for (int p = pair + 1; p <= plast; ++p) {
    const float* slot = P.part + static_cast<size_t>(p * 2 + xi) * P.slot_elems + static_cast<size_t>(cb) * SK_BM +
                        quarter * 32 + c4;
    float4 q[4];
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const int j = i * 4 + jb;
      q[i] = j < ncol ? *reinterpret_cast<const float4*>(slot + j * SK_BM) : make_float4(0.f, 0.f, 0.f, 0.f);
    }
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      w[i].x += q[i].x; w[i].y += q[i].y; w[i].z += q[i].z; w[i].w += q[i].w;
    }
  }
  const size_t o0 = static_cast<size_t>(m0 + cb) * P.ldo + ocol(P, nn);
  if (EPI == EPI_STORE || EPI == EPI_GELU) {
    const bool act = EPI == EPI_GELU && act_on(P, nn) && !(P.dbg_epi & 1);
    bf16* dst = static_cast<bf16*>(P.out) + o0;
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const int j = i * 4 + jb;
      if (j >= ncol || (P.dbg_epi & 2)) continue;
      float4 x = w[i];
      if (act) { x.x = gelu_fast(x.x); x.y = gelu_fast(x.y); x.z = gelu_fast(x.z); x.w = gelu_fast(x.w); }
      __nv_bfloat162 lo = __floats2bfloat162_rn(x.x, x.y), hi = __floats2bfloat162_rn(x.z, x.w);
      *reinterpret_cast<uint2*>(dst + static_cast<size_t>(j) * P.ldo) =
          make_uint2(*reinterpret_cast<uint32_t*>(&lo), *reinterpret_cast<uint32_t*>(&hi));
    }
  } else {
    float* dst = static_cast<float*>(P.out) + o0;
    float4 y[4];
    if (EPI == EPI_ACC_F32) {
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        const int j = i * 4 + jb;
        y[i] = j < ncol ? *reinterpret_cast<const float4*>(dst + static_cast<size_t>(j) * P.ldo) : make_float4(0.f, 0.f, 0.f, 0.f);
      }
    }
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const int j = i * 4 + jb;
      if (j >= ncol) continue;
      float4 x = w[i];
      if (EPI == EPI_ACC_F32) { x.x += y[i].x; x.y += y[i].y; x.z += y[i].z; x.w += y[i].w; }
      *reinterpret_cast<float4*>(dst + static_cast<size_t>(j) * P.ldo) = x;
    }
  }
  __syncwarp();
}

// Lane-per-weight-row final epilogue of one 16-token block (greedy argmax,
// outputs not 16-byte aligned); the owner of a split tile adds the later
// pieces' partials.
template <int EPI>
FL_DEV void rowwise16(const SkParams& P, const uint32_t* r, float bv, float* ws_, int lane, int quarter, int n,
                      bool nok, int nbase, int m0, int cb, int ncol, int pair, int plast, int xi, int row) {
  float v[16];
#pragma unroll
  for (int j = 0; j < 16; ++j) v[j] = __uint_as_float(r[j]) + bv;
  for (int p = pair + 1; p <= plast; ++p) {
    const float* slot = P.part + static_cast<size_t>(p * 2 + xi) * P.slot_elems + cb * SK_BM + row;
    float q[16];
#pragma unroll
    for (int j = 0; j < 16; ++j) q[j] = j < ncol ? slot[j * SK_BM] : 0.f;
#pragma unroll
    for (int j = 0; j < 16; ++j) v[j] += q[j];
  }
  if (EPI == EPI_ARGMAX) {
    // transpose through smem (stride 33: conflict-free both ways) so lane t
    // (< 16) scans token t's 32 weight rows
    float* tb = ws_;
#pragma unroll
    for (int j = 0; j < 16; ++j) tb[j * 33 + lane] = v[j];
    __syncwarp();
    // lane t scans rows 16*(t / 16) .. +15 of token t % 16; the halves combine
    const int nb = nbase + quarter * 32 + 16 * (lane >> 4), tok = lane & 15;
    unsigned long long key = 0ull;
#pragma unroll 8
    for (int cc = 0; cc < 16; ++cc) {
      if (nb + cc < P.N) {
        const unsigned long long k2 = argmax_key(tb[tok * 33 + 16 * (lane >> 4) + cc], P.index_base + nb + cc);
        key = k2 > key ? k2 : key;
      }
    }
    const unsigned long long ko = __shfl_xor_sync(0xffffffffu, key, 16);
    key = ko > key ? ko : key;
    __syncwarp();
    if (lane < ncol && key) atomicMax(&P.keys[m0 + cb + lane], key);
  } else if (nok) {
    const size_t o0 = static_cast<size_t>(m0 + cb) * P.ldo + ocol(P, n);
    const bool act = EPI == EPI_GELU && act_on(P, n);
#pragma unroll
    for (int j = 0; j < 16; ++j) {
      if (j >= ncol) continue;
      const size_t o = o0 + static_cast<size_t>(j) * P.ldo;
      if (EPI == EPI_STORE || EPI == EPI_GELU)
        static_cast<bf16*>(P.out)[o] = __float2bfloat16_rn(act ? gelu_fast(v[j]) : v[j]);
      else if (EPI == EPI_ACC_F32)
        static_cast<float*>(P.out)[o] += v[j];
      else
        static_cast<float*>(P.out)[o] = v[j];
    }
  }
}

template <int EPI>
__global__ void __launch_bounds__(SK_THREADS, 1)
    k_gemm_sk(const __grid_constant__ CUtensorMap tma_w, const __grid_constant__ CUtensorMap tma_x,
              const __grid_constant__ CUtensorMap tma_x2, const __grid_constant__ SkParams P) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  __shared__ __align__(8) uint64_t full_bar[SK_MAXST];
  __shared__ __align__(8) uint64_t empty_bar[SK_MAXST];
  __shared__ __align__(8) uint64_t tfull_bar[SK_MAXBUF];
  __shared__ __align__(8) uint64_t tempty_bar[SK_MAXBUF];
  __shared__ uint32_t tmem_base;
  __shared__ unsigned long long issue_clk[SK_MAXST];   // diagnostics: W issue time per stage
  __shared__ __align__(16) float stg[8 * 16 * SK_STG_LD];   // epilogue transpose, 16x36 per warp

  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  unsigned long long g_start = 0;
  if (P.dbg) asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(g_start));
  // let the next kernel's CTAs launch (and run their prologue) now: it only
  // launches once every CTA of this grid has started, and its
  // griddepcontrol.wait still waits for this grid's completion
  pdl_trigger();
  const int xi = blockIdx.x & 1;                 // position in the pair (cluster rank)
  const int pair = blockIdx.x >> 1;              // pair id = work range
  const bool leader = xi == 0;
  const uint32_t prank = cluster_ctarank() & ~1u;   // the pair's leader in the cluster
  const uint16_t pmask = static_cast<uint16_t>(3u << prank);
  const int XB = (P.bn / 2) * SK_BK * 2;         // this CTA's half of a token sub-tile (64 K)
  const int KPB = P.kpb;                         // 64-wide K sub-chunks per unit
  const int AB = KPB * SK_A_BYTES;               // weight bytes per stage and CTA
  const int STAGE = AB + P.mt * KPB * XB;
  const int stages = P.stages, kch = P.kch;
  const Ranges R = pair_ranges(P, pair);
  const int n0u = R.hi[0] - R.lo[0], nunits = n0u + R.hi[1] - R.lo[1];
  if (P.dbg && threadIdx.x == 0) P.dbg[4 * 9216 + blockIdx.x * 4 + 0] = gtimer();

  if (threadIdx.x == 0) {
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tma_w)) : "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tma_x)) : "memory");
    if (P.nsplit) asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tma_x2)) : "memory");
    for (int s = 0; s < stages; ++s) {
      mbar_init(&full_bar[s], 1 + P.mt);   // weight producer + one per token sub-tile
      mbar_init(&empty_bar[s], 1);           // the pair's MMAs consumed the stage
    }
    for (int b = 0; b < SK_MAXBUF; ++b) {
      mbar_init(&tfull_bar[b], 1);
      mbar_init(&tempty_bar[b], 16);  // 8 epilogue warps x 2 CTAs
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&tmem_base)),
                 "r"(P.ncols));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;");
    if (P.dbg && lane == 0) P.dbg[4 * 9216 + blockIdx.x * 4 + 1] = gtimer();
  }
  if (P.dbg && threadIdx.x == 0) P.dbg[4 * 9216 + blockIdx.x * 4 + 2] = gtimer();
  tc_fence_before();
  cluster_sync_all();
  tc_fence_after();
  if (P.dbg && threadIdx.x == 0) P.dbg[4 * 9216 + blockIdx.x * 4 + 3] = gtimer();
  const uint32_t tmem = tmem_base;
  const int acc_cols = P.mt * P.bn;

  if (warp == 0 || warp == 6 || warp == 7) {
    // producers: warp 0 streams the weight tiles, warp 6 + j the token
    // sub-tile j -- one TMA request per thread per K chunk (a request costs
    // its issuing thread ~250 cycles, tools/probes/tma_rate.cu)
    const int role = warp == 0 ? -1 : warp - 6;   // -1: weights, j >= 0: token sub-tile j
    if (lane == 0 && role < P.mt && role >= -1) {
      const uint32_t my_tx = 2u * (role < 0 ? AB : KPB * XB);   // both CTAs' bytes
      // units are issued strictly in order: walk the coordinates incrementally
      // (divisions only at a tile boundary or the jump to the stream-K range)
      int cur_u = -2, cur_kk = 0, cur_m0 = 0, cur_n0 = 0;
      auto issue = [&](int u, int st) {
        if (u == cur_u + 1 && cur_kk + 1 < kch) {
          ++cur_kk;
        } else {
          const int t = u / kch;
          cur_kk = u - t * kch;
          const int tn = t / P.ntm, tm = t - tn * P.ntm;
          cur_m0 = tm * P.span;
          cur_n0 = tn * 2 * SK_BM + xi * SK_BM;
        }
        cur_u = u;
        const int m0 = cur_m0, n0 = cur_n0, k = cur_kk * SK_BK * KPB;
        const CUtensorMap* xm = P.nsplit && n0 >= P.nsplit ? &tma_x2 : &tma_x;   // dual GEMM: 2nd operand
        // weight coordinates: row-major W -> (k, n0); tiled W -> the first
        // row of the contiguous 128 x 64 chunk (tile n0/128, K chunk k/64)
        const int wcol = P.w_tiled ? 0 : k;
        const int wrow = P.w_tiled ? ((n0 >> 7) * P.kch64 + (k >> 6)) * SK_BM : n0;
        if ((P.dbg_skip_x && role >= 0) || (P.dbg_skip_x == 2 && role < 0)) {   // diagnostic (garbage results)
          if (leader) mbar_expect_tx(&full_bar[st], 0);
          return;
        }
        if (leader) mbar_expect_tx(&full_bar[st], my_tx);
        if (P.dbg && role < 0) issue_clk[st] = clock64();
        if (P.dbg && role == 0 && u < 32 + R.lo[0] && u >= R.lo[0]) P.dbg[4 * 12288 + blockIdx.x * 32 + (u - R.lo[0])] = gtimer();
        if (P.dbg && role < 0 && u < 32 + R.lo[0] && u >= R.lo[0]) P.dbg[4 * 14336 + blockIdx.x * 32 + (u - R.lo[0])] = gtimer();
        if (role < 0 && KPB > 1 && P.w_tiled)
          tma_load_pair(&tma_w, &full_bar[st], smem + st * STAGE, 0, wrow);   // 2 chunks, 32 KB contiguous
        else if (role < 0 && KPB > 1)
          tma_load_pair3(&tma_w, &full_bar[st], smem + st * STAGE, n0, k / SK_BK);
        else if (role >= 0 && KPB > 1)
          tma_load_pair3(xm, &full_bar[st], smem + st * STAGE + AB + role * KPB * XB,
                         m0 + role * P.bn + xi * (P.bn / 2), k / SK_BK);
        else if (role < 0)
          tma_load_pair(&tma_w, &full_bar[st], smem + st * STAGE, wcol, wrow);
        else
          tma_load_pair(xm, &full_bar[st], smem + st * STAGE + AB + role * XB, k,
                        m0 + role * P.bn + xi * (P.bn / 2));
      };
      auto unit = [&](int i) { return i < n0u ? R.lo[0] + i : R.lo[1] + (i - n0u); };
      // L2 prefetch of a unit's weights (no smem): a CTA that starts while its
      // predecessor is still running can only fill its ring, then waits for
      // the activations (griddepcontrol.wait); meanwhile the next units'
      // weights are pulled into L2, so its first stages after the wait land
      // at L2 latency instead of HBM latency
      auto prefetch = [&](int u) {
        const int t = u / kch, kk = u - t * kch;
        const int tn = t / P.ntm;
        const int n0 = tn * 2 * SK_BM + xi * SK_BM, k = kk * SK_BK * KPB;
        if (KPB > 1 && P.w_tiled)
          asm volatile("cp.async.bulk.prefetch.tensor.2d.L2.global.tile [%0, {%1, %2}];" ::"l"(
                           reinterpret_cast<uint64_t>(&tma_w)), "r"(0), "r"(((n0 >> 7) * P.kch64 + (k >> 6)) * SK_BM)
                       : "memory");
        else if (KPB > 1)
          asm volatile("cp.async.bulk.prefetch.tensor.3d.L2.global.tile [%0, {%1, %2, %3}];" ::"l"(
                           reinterpret_cast<uint64_t>(&tma_w)), "r"(0), "r"(n0), "r"(k / SK_BK)
                       : "memory");
        else
          asm volatile("cp.async.bulk.prefetch.tensor.2d.L2.global.tile [%0, {%1, %2}];" ::"l"(
                           reinterpret_cast<uint64_t>(&tma_w)), "r"(P.w_tiled ? 0 : k),
                       "r"(P.w_tiled ? ((n0 >> 7) * P.kch64 + (k >> 6)) * SK_BM : n0)
                       : "memory");
      };
      const int pre = min(nunits, stages);
      if (role >= 0) pdl_wait();            // activations are the predecessor's output
      if (P.dbg && role == 0) P.dbg[4 * (8192 + blockIdx.x) + 0] = gtimer();
      for (int i = 0; i < pre; ++i) issue(unit(i), i);   // weights stream ahead of the wait
      if (role == -1 && P.l2_ahead > 0)
        for (int i = pre; i < min(nunits, pre + P.l2_ahead); ++i) prefetch(unit(i));
      int s = pre % stages;
      uint32_t ph = pre == stages ? 1u : 0u;
      unsigned long long waited = 0, t_start = clock64();
      for (int i = pre; i < nunits; ++i) {
        const unsigned long long tw = P.dbg ? clock64() : 0;
        mbar_wait(&empty_bar[s], ph ^ 1);
        if (P.dbg) waited += clock64() - tw;
        issue(unit(i), s);
        if (++s == stages) { s = 0; ph ^= 1; }
      }
      if (P.dbg && role == -1) {
        P.dbg[4 * blockIdx.x + 0] = waited;
        P.dbg[4 * blockIdx.x + 1] = clock64() - t_start;
      }
    }
    __syncwarp();
  } else if (warp == 1) {
    if (leader) {                          // the whole warp; one elected lane issues
      const uint32_t idesc = idesc_bf16(2 * SK_BM, P.bn);
      int s = 0, seg = 0;
      uint32_t ph = 0;
      unsigned long long waited = 0, twait = 0, lat = 0, nlat = 0, t_start = clock64();
      for (int r = 0; r < 2; ++r)
      for (int u = R.lo[r]; u < R.hi[r];) {
        const Seg g = seg_at(u, R.hi[r], kch);
        const int klo = g.klo, khi = g.khi;
        const int b = seg % P.nbuf;
        const uint32_t use = static_cast<uint32_t>(seg / P.nbuf);
        unsigned long long tw = P.dbg ? clock64() : 0;
        mbar_wait(&tempty_bar[b], (use & 1) ^ 1);   // epilogue drained this buffer
        if (P.dbg) twait += clock64() - tw;
        tc_fence_after();
        const uint32_t acc = tmem + b * acc_cols;
        for (int c = klo; c < khi; ++c) {
          tw = P.dbg ? clock64() : 0;
          mbar_wait(&full_bar[s], ph);
          if (P.dbg && nlat < 32) P.dbg[4 * 10240 + blockIdx.x * 32 + nlat] = gtimer();
          if (P.dbg) {
            const unsigned long long now = clock64();
            waited += now - tw;
            lat += now - *reinterpret_cast<volatile unsigned long long*>(&issue_clk[s]);
            ++nlat;
          }
          tc_fence_after();
          const uint8_t* st = smem + s * STAGE;
          if (KPB == 2 && P.mt == 1 && !P.dbg_skip_mma) {
            static_assert(SK_A_BYTES == 16384, "mma_stage2_elect steps A by 16 KB");
            mma_stage2_elect(acc, desc_sw128(st), desc_sw128(st + AB), desc_sw128(st + AB + XB), idesc,
                             c > klo ? 1u : 0u);
            commit_pair_elect(&empty_bar[s], pmask);
            if (++s == stages) { s = 0; ph ^= 1; }
            continue;
          }
          for (int kc = 0; kc < KPB && !P.dbg_skip_mma; ++kc) {
            const uint64_t ad = desc_sw128(st + kc * SK_A_BYTES);
            if (P.mt == 2) {
              // consecutive MMAs share the weight slab (A) across the two token sub-tiles
              const uint64_t bd0 = desc_sw128(st + AB + kc * XB), bd1 = desc_sw128(st + AB + (KPB + kc) * XB);
#pragma unroll
              for (int kk = 0; kk < SK_BK / 16; ++kk) {
                mma_pair_elect(acc, ad + 2 * kk, bd0 + 2 * kk, idesc, (c > klo) | kc | kk);
                mma_pair_elect(acc + P.bn, ad + 2 * kk, bd1 + 2 * kk, idesc, (c > klo) | kc | kk);
              }
              continue;
            }
            for (int j = 0; j < P.mt; ++j) {
              const uint64_t bd = desc_sw128(st + AB + (j * KPB + kc) * XB);
#pragma unroll
              for (int kk = 0; kk < SK_BK / 16; ++kk)
                mma_pair_elect(acc + j * P.bn, ad + 2 * kk, bd + 2 * kk, idesc, (c > klo) | kc | kk);
            }
          }
          commit_pair_elect(&empty_bar[s], pmask);
          if (++s == stages) { s = 0; ph ^= 1; }
        }
        commit_pair_elect(&tfull_bar[b], pmask);
        u += khi - klo;
        ++seg;
      }
      if (P.dbg && lane == 0) {
        P.dbg[4 * (8192 + blockIdx.x) + 1] = gtimer();
        P.dbg[4 * blockIdx.x + 2] = waited;
        P.dbg[4 * blockIdx.x + 3] = clock64() - t_start;
        P.dbg[4 * (2048 + blockIdx.x) + 0] = twait;
        P.dbg[4 * (2048 + blockIdx.x) + 1] = nlat ? lat / nlat : 0;
      }
    }
  } else {
    // ---------------------------------------------------------------- epilogue
    // warps 2-5 and 8-11: a warp reads TMEM lane quarter warp % 4; the two
    // warps of a quarter take alternate 16-token blocks (the epilogue, not
    // the weight stream, bounds the wide windows: profiles/r02b_*)
    pdl_wait();   // EPI_ACC_F32 reads `out`, written by predecessors
    const int quarter = warp & 3, half = warp >= 8 ? 1 : 0;
    float* ws_ = stg + (half * 4 + quarter) * (16 * SK_STG_LD);
    const int row = quarter * 32 + lane;
    int seg = 0;
    unsigned long long e_wait = 0, e_flag = 0, e_blk = 0, e_post = 0, e_ld = 0, e_sts = 0, e_t0 = clock64();
    if (P.csplit > 1) {
      // ---- even split-K: the S pairs t*S .. t*S+S-1 each hold the fp32 partial
      // of one K piece of tile t.  All publish, then piece s reduces tokens
      // [s, s+1) * mcount / S over the S slots and runs the epilogue -- the
      // fix-up is spread over the S pairs instead of serialised in one owner.
      const int S = P.csplit;
      const int t = R.lo[0] / kch, piece = pair - t * S;
      const int tn = t / P.ntm, tm = t - tn * P.ntm;
      const int m0 = tm * P.span;
      const int mcount = min(P.slice, P.M - m0);
      const int nbase = tn * 2 * SK_BM + xi * SK_BM;
      const uint32_t tacc = tmem + (static_cast<uint32_t>(quarter * 32) << 16);
      if (warp == 2 && lane == 0) mbar_wait_sleep(&tfull_bar[0], 0);
      epi_bar();
      tc_fence_after();
      float* pub = P.part + static_cast<size_t>(pair * 2 + xi) * P.slot_elems;
      for (int cb = 16 * half; cb < mcount; cb += 32) {
        uint32_t r[16];
        tmem_ld16(tacc + cb, r);
        block16<EPI, BLK_PUB>(P, r, 0.f, ws_, lane, quarter, nbase, m0, cb, min(16, mcount - cb), pub);
      }
      // publish -> arrive: the CTA barrier orders every thread's partial
      // stores before one thread's gpu-scope release (CUTLASS's semaphore
      // pattern; a __threadfence in every thread costs ~1 us here)
      const unsigned long long tf0 = P.dbg ? clock64() : 0;
      epi_bar();
      unsigned* arrive = P.flags + 2 * SK_MAX_PAIRS + (t * 2 + xi);
      unsigned* done = arrive + 2 * SK_MAX_PAIRS;
      if (warp == 2 && lane == 0) {
        red_release_add(arrive, 1u);
        long long spins = 0;
        while (ld_acquire(arrive) < static_cast<unsigned>(S)) {
          __nanosleep(32);
          if (++spins > (1ll << 26)) __trap();
        }
      }
      epi_bar();
      if (P.dbg) e_flag += clock64() - tf0;
      // reduce my token slice: warp takes tokens, lane = 4 weight rows.  The
      // partials come from L2 (other SMs wrote them): UN tokens' loads (x S
      // pieces, + the residual for ACC) are issued before any is used
      const int lo = piece * mcount / S, hi = (piece + 1) * mcount / S;
      const int rrow = lane * 4;                      // row within this CTA's 128
      const int nn = nbase + rrow;
      float b4[4] = {0.f, 0.f, 0.f, 0.f};
      if (P.bias)
        for (int q = 0; q < 4; ++q) b4[q] = nn + q < P.N ? __bfloat162float(P.bias[nn + q]) : 0.f;
      const bool act = EPI == EPI_GELU && act_on(P, nn);
      const bool v4 = nn + 3 < P.N && P.vec;
      const float* slot0 = P.part + static_cast<size_t>((t * S) * 2 + xi) * P.slot_elems + rrow;
      const size_t pstride = static_cast<size_t>(2) * P.slot_elems;   // next piece's slot
      constexpr int UN = 4;
      const int ew = half * 4 + quarter;
      for (int tok0 = lo + ew; tok0 < hi; tok0 += 8 * UN) {
        float4 q[UN][4];
        float4 y[UN];
#pragma unroll
        for (int u = 0; u < UN; ++u) {
          const int tok = tok0 + 8 * u;
#pragma unroll
          for (int p = 0; p < 4; ++p)
            q[u][p] = (p < S && tok < hi) ? *reinterpret_cast<const float4*>(slot0 + p * pstride + static_cast<size_t>(tok) * SK_BM)
                                          : make_float4(0.f, 0.f, 0.f, 0.f);
          y[u] = make_float4(0.f, 0.f, 0.f, 0.f);
          if (EPI == EPI_ACC_F32 && v4 && tok < hi)
            y[u] = *reinterpret_cast<const float4*>(static_cast<float*>(P.out) + static_cast<size_t>(m0 + tok) * P.ldo + nn);
        }
#pragma unroll
        for (int u = 0; u < UN; ++u) {
          const int tok = tok0 + 8 * u;
          if (tok >= hi) break;
          float4 acc = make_float4(b4[0], b4[1], b4[2], b4[3]);
#pragma unroll
          for (int p = 0; p < 4; ++p) {
            acc.x += q[u][p].x; acc.y += q[u][p].y; acc.z += q[u][p].z; acc.w += q[u][p].w;
          }
          const size_t o = static_cast<size_t>(m0 + tok) * P.ldo + ocol(P, nn);
          if (v4) {
            if (EPI == EPI_ACC_F32) {
              *reinterpret_cast<float4*>(static_cast<float*>(P.out) + o) =
                  make_float4(y[u].x + acc.x, y[u].y + acc.y, y[u].z + acc.z, y[u].w + acc.w);
            } else if (EPI == EPI_STORE_F32) {
              *reinterpret_cast<float4*>(static_cast<float*>(P.out) + o) = acc;
            } else {
              if (act) {
                acc.x = gelu_fast(acc.x); acc.y = gelu_fast(acc.y); acc.z = gelu_fast(acc.z); acc.w = gelu_fast(acc.w);
              }
              __nv_bfloat162 l2 = __floats2bfloat162_rn(acc.x, acc.y), h2 = __floats2bfloat162_rn(acc.z, acc.w);
              *reinterpret_cast<uint2*>(static_cast<bf16*>(P.out) + o) =
                  make_uint2(*reinterpret_cast<uint32_t*>(&l2), *reinterpret_cast<uint32_t*>(&h2));
            }
          } else {
            const float a4[4] = {acc.x, acc.y, acc.z, acc.w};
            for (int qq = 0; qq < 4 && nn + qq < P.N; ++qq) {
              if (EPI == EPI_ACC_F32) static_cast<float*>(P.out)[o + qq] += a4[qq];
              else if (EPI == EPI_STORE_F32) static_cast<float*>(P.out)[o + qq] = a4[qq];
              else static_cast<bf16*>(P.out)[o + qq] = __float2bfloat16_rn(act ? gelu_fast(a4[qq]) : a4[qq]);
            }
          }
        }
      }
      epi_bar();
      if (warp == 2 && lane == 0) {
        // the last reader re-arms both counters for the next launch
        if (atomicAdd(done, 1u) == static_cast<unsigned>(S - 1)) {
          *arrive = 0u;
          *done = 0u;
          __threadfence();
        }
      }
      tc_fence_before();
    }
    for (int r = 0; r < 2 && P.csplit == 1; ++r)
    for (int u = R.lo[r]; u < R.hi[r];) {
      const Seg g = seg_at(u, R.hi[r], kch);
      const int t = g.t, klo = g.klo, khi = g.khi;
      const int b = seg % P.nbuf;
      const uint32_t use = static_cast<uint32_t>(seg / P.nbuf);
      const int tn = t / P.ntm, tm = t - tn * P.ntm;
      const int m0 = tm * P.span;
      const int mcount = min(P.slice, P.M - m0);
      const int nbase = tn * 2 * SK_BM + xi * SK_BM;
      const int n = nbase + row;
      const bool nok = n < P.N;
      const bool whole = klo == 0 && khi == kch;
      const float bv = (P.bias && nok && klo == 0) ? __bfloat162float(P.bias[n]) : 0.f;
      const uint32_t tacc = tmem + (static_cast<uint32_t>(quarter * 32) << 16) + b * acc_cols;
      unsigned long long tw0 = P.dbg ? clock64() : 0;
      if (warp == 2 && lane == 0) mbar_wait_sleep(&tfull_bar[b], use & 1);
      epi_bar();
      if (P.dbg) e_wait += clock64() - tw0;
      if (P.dbg && warp == 2 && lane == 0 && seg == 0) P.dbg[4 * (8192 + blockIdx.x) + 2] = gtimer();
      tc_fence_after();
      if (P.dbg_skip_epi == 1) {   // diagnostic: skip epilogue work
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive_cluster(&tempty_bar[b], prank);
        u += khi - klo;
        ++seg;
        continue;
      }

      // segment mode: final epilogue (whole tile, or the k = 0 owner of a split
      // tile after folding in the later pieces), publish (a later piece of a
      // split tile: the first segment of its pair's stream-K range) or red
      // (a piece of a split residual tile)
      int mode = BLK_FINAL, plast = pair;      // plast: last pair holding a piece
      if (!whole && EPI == EPI_ACC_F32 && P.red) {
        mode = BLK_RED;
      } else if (!whole) {
        if (klo > 0) {
          mode = BLK_PUB;
        } else {
          plast = owner_of((t + 1) * kch - 1, P);
          const unsigned long long tf0 = P.dbg ? clock64() : 0;
          if (warp == 2 && lane == 0) {
            for (int q = pair + 1; q <= plast; ++q) {
              const unsigned* f = &P.flags[q * 2 + xi];
              long long spins = 0;
              while (ld_acquire(f) == 0u) {
                __nanosleep(64);
                if (++spins > (1ll << 26)) __trap();   // a lost partial: fail loudly, never hang
              }
            }
          }
          epi_bar();
          if (P.dbg) e_flag += clock64() - tf0;
        }
      }
      float* pub = P.part + static_cast<size_t>(pair * 2 + xi) * P.slot_elems;
      const unsigned long long tb0 = P.dbg ? clock64() : 0;
      // Each mode has its own loop (mixing them lets the compiler predicate the
      // loads / atomics of other modes into the hot loop: 6x slower).  Stores
      // go through a per-warp smem transpose so every lane moves 16 bytes
      // (4 weight rows of one token, tools/probes/store_probe.cu: 2.8x).
      const bool vec = P.vec && nbase + SK_BM <= P.N;
      if (mode == BLK_PUB) {
        for (int cb = 16 * half; cb < mcount; cb += 32) {
          uint32_t r[16];
          tmem_ld16(tacc + cb, r);
          block16<EPI, BLK_PUB>(P, r, bv, ws_, lane, quarter, nbase, m0, cb, min(16, mcount - cb), pub);
        }
      } else if (EPI == EPI_ACC_F32 && mode == BLK_RED && vec) {
        for (int cb = 16 * half; cb < mcount; cb += 32) {
          uint32_t r[16];
          tmem_ld16(tacc + cb, r);
          block16<EPI, BLK_RED>(P, r, bv, ws_, lane, quarter, nbase, m0, cb, min(16, mcount - cb), pub);
        }
      } else if (EPI == EPI_ACC_F32 && mode == BLK_RED) {
        // unaligned residual rows: scalar float atomics, lane = weight row
        for (int cb = 16 * half; cb < mcount; cb += 32) {
          uint32_t r[16];
          tmem_ld16(tacc + cb, r);
          const int ncol = min(16, mcount - cb);
          if (nok) {
            float* dst = static_cast<float*>(P.out) + static_cast<size_t>(m0 + cb) * P.ldo + n;
#pragma unroll
            for (int j = 0; j < 16; ++j)
              if (j < ncol) atomicAdd(dst + static_cast<size_t>(j) * P.ldo, __uint_as_float(r[j]) + bv);
          }
        }
      } else if (EPI == EPI_ARGMAX || !vec) {
        for (int cb = 16 * half; cb < mcount; cb += 32) {
          uint32_t r[16];
          tmem_ld16(tacc + cb, r);
          rowwise16<EPI>(P, r, bv, ws_, lane, quarter, n, nok, nbase, m0, cb, min(16, mcount - cb), pair, plast, xi,
                         row);
        }
      } else {
        for (int cb = 16 * half; cb < mcount; cb += 32) {
          uint32_t r[16];
          const unsigned long long tl0 = P.dbg ? clock64() : 0;
          tmem_ld16(tacc + cb, r);
          if (P.dbg) e_ld += clock64() - tl0;
          final16<EPI>(P, r, bv, ws_, lane, quarter, nbase, m0, cb, min(16, mcount - cb), pair, plast, xi);
        }
      }
      const unsigned long long tb1 = P.dbg ? clock64() : 0;
      if (P.dbg) e_blk += tb1 - tb0;
      if (mode == BLK_PUB) {
        epi_bar();      // every thread's partial stores before the release
        if (warp == 2 && lane == 0) st_release(&P.flags[pair * 2 + xi], 1u);
      } else if (plast > pair) {
        epi_bar();
        if (warp == 2 && lane == 0)
          for (int q = pair + 1; q <= plast; ++q) P.flags[q * 2 + xi] = 0u;   // re-arm
      }
      // this buffer may be overwritten by the next-but-(nbuf-1) segment --
      // unless this was the pair's last segment (no MMA waits on it; the
      // release-ordered remote arrive would wait for this warp's stores:
      // out-projection at 16 / 144 rows 761 -> 752 / 882 -> 873 us per 28
      // layers, C2 step 491 -> 483 us)
      const bool last_seg = u + (khi - klo) >= R.hi[r] && (r == 1 || R.hi[1] <= R.lo[1]);
      tc_fence_before();
      __syncwarp();
      if (lane == 0 && !last_seg) mbar_arrive_cluster(&tempty_bar[b], prank);
      if (P.dbg) e_post += clock64() - tb1;
      u += khi - klo;
      ++seg;
    }
    if (P.dbg && warp == 2 && lane == 0) {
      unsigned long long g_end;
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(g_end));
      P.dbg[4 * (4096 + blockIdx.x) + 0] = g_start;
      P.dbg[4 * (4096 + blockIdx.x) + 1] = g_end;
      P.dbg[4 * (4096 + blockIdx.x) + 2] = e_wait;
      P.dbg[4 * (4096 + blockIdx.x) + 3] = clock64() - e_t0;
      P.dbg[4 * (6144 + blockIdx.x) + 0] = e_flag;
      P.dbg[4 * (6144 + blockIdx.x) + 1] = e_blk;
      P.dbg[4 * (6144 + blockIdx.x) + 2] = e_post;
      P.dbg[4 * (6144 + blockIdx.x) + 3] = e_ld;
      P.dbg[4 * (4096 + blockIdx.x) + 3] = e_sts;
    }
  }

  __syncwarp();
  tc_fence_before();
  __syncwarp();
  // the pair's TMEM is freed jointly.  Only TMEM is handed over here and its
  // accesses are ordered by the tcgen05 fences around this execution
  // barrier, so the arrive is relaxed: a release would first drain every
  // thread's epilogue stores (C2 step 484 -> 472 us)
  asm volatile("barrier.cluster.arrive.relaxed.aligned;\n\tbarrier.cluster.wait.aligned;" ::: "memory");
  if (warp == 1) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(P.ncols));
    if (P.dbg && threadIdx.x == 32) P.dbg[4 * (8192 + blockIdx.x) + 3] = gtimer();
  }
}

// ------------------------------------------------------------------ host side
PFN_cuTensorMapEncodeTiled_v12000 g_encode_sk = nullptr;

struct MapKey {
  const void* ptr;
  int dtype;               // 0 bf16, 1 f32
  uint64_t rows, cols, ld_bytes;
  uint32_t box_c, box_r;
  int swz;
  int kpb;                 // > 1: 3-D view [cols/64][rows][64], box {64, box_r, kpb}
  bool operator<(const MapKey& o) const {
    return std::tie(ptr, dtype, rows, cols, ld_bytes, box_c, box_r, swz, kpb) <
           std::tie(o.ptr, o.dtype, o.rows, o.cols, o.ld_bytes, o.box_c, o.box_r, o.swz, o.kpb);
  }
};
std::map<MapKey, CUtensorMap> g_sk_maps;

// 2-D row-major tensor [rows][cols] (row stride ld_bytes), box [box_r][box_c]
bool sk_map(const MapKey& key, CUtensorMap** out) {
  auto it = g_sk_maps.find(key);
  if (it != g_sk_maps.end()) {
    *out = &it->second;
    return true;
  }
  if (!g_encode_sk) {
    cudaDriverEntryPointQueryResult q;
    void* fn = nullptr;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q) != cudaSuccess || !fn) {
      g_sk_err = "cuTensorMapEncodeTiled entry point unavailable";
      return false;
    }
    g_encode_sk = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fn);
  }
  CUtensorMap map;
  const bool d3 = key.kpb > 1;
  cuuint64_t dims[3] = {d3 ? 64 : key.cols, key.rows, key.cols / 64};
  cuuint64_t strides[2] = {key.ld_bytes, 128};
  cuuint32_t box[3] = {key.box_c, key.box_r, static_cast<cuuint32_t>(key.kpb)};
  cuuint32_t estr[3] = {1, 1, 1};
  CUresult r = g_encode_sk(&map, key.dtype ? CU_TENSOR_MAP_DATA_TYPE_FLOAT32 : CU_TENSOR_MAP_DATA_TYPE_BFLOAT16,
                           d3 ? 3 : 2, const_cast<void*>(key.ptr), dims, strides, box, estr,
                           CU_TENSOR_MAP_INTERLEAVE_NONE,
                           key.swz ? CU_TENSOR_MAP_SWIZZLE_128B : CU_TENSOR_MAP_SWIZZLE_NONE,
                           CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) {
    char buf[160];
    snprintf(buf, sizeof buf, "cuTensorMapEncodeTiled failed (%d) rows=%llu cols=%llu", (int)r,
             (unsigned long long)key.rows, (unsigned long long)key.cols);
    g_sk_err = buf;
    return false;
  }
  *out = &(g_sk_maps[key] = map);
  return true;
}

}  // namespace

size_t sk_workspace_bytes() {
  return (size_t)SK_MAX_PAIRS * 2 * SK_MAX_SPAN * SK_BM * 4 + SK_MAX_PAIRS * 6 * 4 + 256;
}

const char* sk_last_error() { return g_sk_err.c_str(); }
void sk_tune(int key, int value) {
  if (key >= 1 && key < 10) g_tune[key] = value;
  if (key == 8) g_l2_ahead = value;
}
void sk_set_debug(unsigned long long* p) { g_sk_dbg = p; }

int sk_init(void* base, size_t bytes) {
  if (bytes < sk_workspace_bytes()) {
    g_sk_err = "stream-K workspace too small";
    return -1;
  }
  // flags live after the partial slots and must start at zero (self-resetting after)
  char* f = static_cast<char*>(base) + (size_t)SK_MAX_PAIRS * 2 * SK_MAX_SPAN * SK_BM * 4;
  if (cudaMemset(f, 0, SK_MAX_PAIRS * 6 * 4) != cudaSuccess) {
    g_sk_err = "stream-K flag reset failed";
    return -1;
  }
  return 0;
}

cudaError_t sk_rearm(void* base, cudaStream_t s) {
  char* f = static_cast<char*>(base) + (size_t)SK_MAX_PAIRS * 2 * SK_MAX_SPAN * SK_BM * 4;
  return cudaMemsetAsync(f, 0, SK_MAX_PAIRS * 6 * 4, s);
}

int gemm_sk(void* ws, int num_sms, const GemmArgs& a, cudaStream_t s) {
  if (a.M <= 0 || a.N <= 0) return 0;
  if (a.dtype != FL_DTYPE_BF16 || a.K % SK_BK || a.ldx % 8) {
    g_sk_err = "tensor-core GEMM needs bf16, K % 64 == 0 and 16-byte aligned rows";
    return -1;
  }
  if (a.nsplit && (a.epi != EPI_GELU || a.nsplit % (2 * SK_BM) || a.nsplit >= a.N || a.ogap < 0)) {
    g_sk_err = "dual GEMM needs EPI_GELU and a split at a multiple of 256 weight rows";
    return -1;
  }
  static bool configured = false;
  if (!configured) {
    for (auto k : {k_gemm_sk<EPI_STORE>, k_gemm_sk<EPI_GELU>, k_gemm_sk<EPI_ACC_F32>, k_gemm_sk<EPI_STORE_F32>,
                   k_gemm_sk<EPI_ARGMAX>})
      cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, SK_RING_BUDGET + 1024);
    configured = true;
  }
  SkParams P{};
  P.M = a.M;
  P.N = a.N;
  P.ldo = a.ldo;
  P.epi = a.epi;
  P.ntn = (a.N + 2 * SK_BM - 1) / (2 * SK_BM);
  // token tiling: the whole window (<= 512 tokens) in one pair, as 1-2 UMMA
  // N sub-tiles, so every weight byte is read once
  // windows wider than span_cap tokens run as several token tiles; tiles are
  // numbered weight-tile-major (t = tn * ntm + tm), so the token tiles of one
  // weight tile are adjacent units (their second weight read can hit L2).
  // Measured (tools/step_gemm_bench.py, C3 shapes): a cap of 256 tokens with
  // double-buffered accumulators is 1.2-1.3x SLOWER at 288-512 rows than the
  // whole window (<= 512) as one token tile -- the default
  const int span_cap = g_tune[5] > 0 ? g_tune[5] : SK_MAX_SPAN;
  const int ntm = (a.M + span_cap - 1) / span_cap;
  const int per = (a.M + ntm - 1) / ntm;                   // tokens per token tile
  P.mt = per <= 256 ? 1 : 2;
  P.bn = (((per + P.mt - 1) / P.mt) + 15) / 16 * 16;
  if (ntm > 1) P.bn = (P.bn + 31) / 32 * 32;               // 32-token epilogue blocks never cross tiles
  P.slice = P.mt * P.bn;
  P.span = P.slice;
  // two 64-wide K sub-chunks per unit (one request per operand) when the
  // deeper stage still leaves >= 3 ring stages: a TMA request costs a roughly
  // fixed time, so bigger boxes stream faster (tools/step_gemm_bench.py,
  // merged out-projection at 192 / 256 rows: 1462 -> 1302 / 1548 -> 1435 us
  // per 28 layers with 3 stages of 64 KB instead of 6 of 32 KB)
  P.kpb = 1;
  {
    const int st2 = 2 * (SK_A_BYTES + P.mt * (P.bn / 2) * SK_BK * 2);
    if (a.K % (2 * SK_BK) == 0 && SK_RING_BUDGET / st2 >= 3) P.kpb = 2;
    if (g_tune[3] == 1 || (g_tune[3] == 2 && a.K % (2 * SK_BK) == 0 && SK_RING_BUDGET / st2 >= 2)) P.kpb = g_tune[3];
  }
  P.kch = a.K / (SK_BK * P.kpb);
  const int stage = P.kpb * (SK_A_BYTES + P.mt * (P.bn / 2) * SK_BK * 2);
  P.stages = SK_RING_BUDGET / stage;
  if (P.stages > SK_MAXST) P.stages = SK_MAXST;
  if (g_tune[2] > 1 && g_tune[2] < P.stages) P.stages = g_tune[2];
  // TMEM accumulator buffers: as many (<= SK_MAXBUF) as fit 512 columns, so
  // the epilogue of a segment may lag the MMAs of the next ones
  {
    const int slice_cols = P.slice <= 32 ? 32 : P.slice <= 64 ? 64 : P.slice <= 128 ? 128 : P.slice;
    int nb = 512 / slice_cols;
    if (g_tune[7] >= 10) nb = g_tune[7] - 10;              // diagnostic: fixed buffer count
    P.nbuf = nb < 1 ? 1 : nb > SK_MAXBUF ? SK_MAXBUF : nb;
  }
  const int cols = P.nbuf * P.slice;
  P.ncols = cols <= 32 ? 32 : cols <= 64 ? 64 : cols <= 128 ? 128 : cols <= 256 ? 256 : 512;
  P.units = ntm * P.ntn * P.kch;
  P.ntm = ntm;
  void (*kern)(const CUtensorMap, const CUtensorMap, const CUtensorMap, const SkParams) = nullptr;
  switch (a.epi) {
    case EPI_STORE: kern = k_gemm_sk<EPI_STORE>; break;
    case EPI_GELU: kern = k_gemm_sk<EPI_GELU>; break;
    case EPI_ACC_F32: kern = k_gemm_sk<EPI_ACC_F32>; break;
    case EPI_STORE_F32: kern = k_gemm_sk<EPI_STORE_F32>; break;
    case EPI_ARGMAX: kern = k_gemm_sk<EPI_ARGMAX>; break;
    default: g_sk_err = "unknown epilogue"; return -1;
  }
  const int smem = P.stages * stage + 1024;
  int npairs = num_sms / 2;
  if (npairs > SK_MAX_PAIRS) npairs = SK_MAX_PAIRS;
  // a persistent grid must be co-resident: pairs of ~200 KB CTAs only fit
  // where a GPC still has 2 free SMs, so ask the occupancy calculator
  {
    static std::map<std::tuple<const void*, int>, int> occ_cache;
    const auto key = std::make_tuple(reinterpret_cast<const void*>(kern), smem);
    auto it = occ_cache.find(key);
    if (it == occ_cache.end()) {
      cudaLaunchConfig_t cfg = {};
      cfg.gridDim = dim3(2 * 128);
      cfg.blockDim = dim3(SK_THREADS);
      cfg.dynamicSmemBytes = smem;
      cudaLaunchAttribute at;
      at.id = cudaLaunchAttributeClusterDimension;
      at.val.clusterDim.x = 2;
      at.val.clusterDim.y = 1;
      at.val.clusterDim.z = 1;
      cfg.attrs = &at;
      cfg.numAttrs = 1;
      int nc = 0;
      if (cudaOccupancyMaxActiveClusters(&nc, kern, &cfg) != cudaSuccess || nc < 1) {
        cudaGetLastError();
        nc = npairs;
      }
      it = occ_cache.emplace(key, nc).first;
    }
    if (npairs > it->second) npairs = it->second;
  }
  if (g_tune[1] > 0 && g_tune[1] < npairs) npairs = g_tune[1];
  // Work decomposition (pair_ranges):
  // * more tiles than pairs: every pair takes the same number of whole tiles
  //   first (no fix-up), the remaining tiles are dealt out stream-K, so all
  //   SMs stream equal weight bytes (merged QKV + FFN-up, LM head, wide
  //   windows);
  // * at most half as many tiles as pairs (attn-out / FFN-down, 16 tiles):
  //   even split-K over S <= 4 pairs per tile with a spread reduction, so the
  //   accumulator is never held for a mid-range fix-up;
  // * otherwise (narrow windows, HBM-bound): stream-K over all pairs.
  const int tiles = ntm * P.ntn;
  P.csplit = 1;
  P.dpw = 0;
  const bool direct = a.epi == EPI_ACC_F32 || a.epi == EPI_STORE_F32 || a.epi == EPI_STORE || a.epi == EPI_GELU;
  // split residual tiles always red.add (no fix-up waits for EPI_ACC_F32)
  P.red = (a.epi == EPI_ACC_F32 && !a.indep) ? 1 : 0;
  if (a.indep) {
    // one whole tile per pair and no fix-up anywhere: correct whatever part
    // of the grid is resident (another stream's kernels may hold SMs)
    npairs = tiles;
    P.dpw = 1;
  } else if (tiles >= npairs) {
    P.dpw = tiles / npairs;
  } else if (a.epi == EPI_ACC_F32) {
    // residual GEMMs (attn-out / FFN-down, 16 tiles): pure stream-K over all
    // pairs, every piece of a split tile red.adds into the fp32 residual --
    // no fix-up, no waits, all 148 SMs stream equal weight bytes
  } else if (a.M >= 64 && direct && 2 * tiles <= npairs && P.kch >= 2) {
    P.csplit = npairs / tiles > 4 ? 4 : npairs / tiles;
    if (P.csplit > P.kch) P.csplit = P.kch;                // every piece holds >= 1 K unit
    npairs = tiles * P.csplit;
  } else if (a.M >= 64) {
    // wide windows: even pieces with owner fix-up beat a ragged stream-K split
    npairs = tiles * min(npairs / tiles, P.kch);
  } else if (a.K <= 1024) {
    // short K (GPT-2 class): a few whole tiles beat the fix-up of a split
    // (the fixed cost per launch dominates)
    npairs = tiles;
  } else {
    const int mu = g_tune[4] > 0 ? g_tune[4] : 4;
    const int cap = (P.units + mu - 1) / mu;               // >= 4 units per range
    if (npairs > cap) npairs = cap;
  }
  if (npairs < 1) npairs = 1;
  P.npairs = npairs;
  {
    // stream-K share of the units after the whole-tile prefix: every range
    // non-empty, and >= 2 units per range behind a prefix
    const int ur = P.units - P.dpw * P.kch * npairs;
    int nsk = P.dpw ? ur / (g_tune[4] > 0 ? g_tune[4] : 2) : ur;
    if (nsk > npairs) nsk = npairs;
    P.nsk = nsk < 1 ? 1 : nsk;
  }
  P.bias = static_cast<const bf16*>(a.bias);
  P.out = a.out;
  P.keys = a.keys;
  P.index_base = a.index_base;
  P.part = static_cast<float*>(ws);
  P.slot_elems = SK_MAX_SPAN * SK_BM;
  P.flags = reinterpret_cast<unsigned*>(static_cast<char*>(ws) + (size_t)SK_MAX_PAIRS * 2 * SK_MAX_SPAN * SK_BM * 4);
  // diagnostics (key 9 = 1): consecutive launches alternate between two
  // 64 K-entry halves of the buffer, so a tool sees a launch and its predecessor
  static unsigned dbg_flip = 0;
  P.dbg = g_sk_dbg && g_tune[9] == 1 ? g_sk_dbg + (dbg_flip++ & 1u) * (4 * 16384) : g_sk_dbg;
  P.dbg_skip_x = g_tune[6] == 1 || g_tune[6] == 2 ? g_tune[6] : 0;   // 2: no weight loads either
  P.dbg_skip_mma = g_tune[7] == 1 ? 1 : 0;   // (key 7 >= 10: TMEM buffer count - 10)
  // key 8 >= 0: L2 prefetch depth (measured: 4..32 units slow every M, so 0);
  // diagnostics: -2 no epilogue, -3 no epilogue for the last segment,
  // -10 - bits: 1 no GELU, 2 no output stores
  P.l2_ahead = g_l2_ahead >= 0 ? g_l2_ahead : 0;
  P.dbg_skip_epi = g_l2_ahead == -2 ? 1 : g_l2_ahead == -3 ? 2 : 0;
  P.dbg_epi = g_l2_ahead <= -10 && g_l2_ahead > -20 ? -10 - g_l2_ahead : 0;
  P.nsplit = a.nsplit;
  P.ogap = a.ogap;
  P.vec = (a.ldo % 4 == 0 && (reinterpret_cast<uintptr_t>(a.out) & 15) == 0) ? 1 : 0;
  CUtensorMap *mw, *mx;
  P.w_tiled = a.w_tiled;
  P.kch64 = a.K / SK_BK;
  if (a.w_tiled) {
    // [rows = ceil(N/128) * 128 * K/64][64]: 128-byte rows, contiguous chunks
    const uint64_t trows = (uint64_t)((a.N + SK_BM - 1) / SK_BM) * SK_BM * (a.K / SK_BK);
    const uint32_t box = P.kpb > 1 ? 2 * SK_BM : (uint32_t)SK_BM;
    if (!sk_map({a.w, 0, trows, (uint64_t)SK_BK, (uint64_t)SK_BK * 2, SK_BK, box, 1, 1}, &mw)) return -1;
  } else if (!sk_map({a.w, 0, (uint64_t)a.N, (uint64_t)a.K, (uint64_t)a.K * 2, SK_BK, (uint32_t)SK_BM, 1, P.kpb},
                     &mw)) {
    return -1;
  }
  if (!sk_map({a.x, 0, (uint64_t)(a.mcap > a.M ? a.mcap : a.M), (uint64_t)a.K, (uint64_t)a.ldx * 2, SK_BK,
               (uint32_t)(P.bn / 2), 1, P.kpb}, &mx))
    return -1;
  CUtensorMap* mx2 = mx;
  if (a.x2 && a.x2 != a.x &&
      !sk_map({a.x2, 0, (uint64_t)(a.mcap > a.M ? a.mcap : a.M), (uint64_t)a.K, (uint64_t)a.ldx * 2, SK_BK,
               (uint32_t)(P.bn / 2), 1, P.kpb}, &mx2))
    return -1;
  cudaError_t e = launch_k(kern, dim3(2 * P.npairs), dim3(SK_THREADS), smem, s, dim3(2, 1, 1), *mw, *mx, *mx2, P);
  if (e != cudaSuccess) {
    char buf[256];
    snprintf(buf, sizeof buf, "k_gemm_sk launch (pairs %d smem %d stages %d bn %d mt %d): %s", P.npairs, smem,
             P.stages, P.bn, P.mt, cudaGetErrorString(e));
    g_sk_err = buf;
    return -1;
  }
  return 0;
}

// ---- the TcWorkspace interface (gemm_tc.cuh) over the stream-K kernel
size_t tc_workspace_bytes(int, int) { return sk_workspace_bytes(); }
const char* tc_last_error() { return sk_last_error(); }
void tc_set_debug(unsigned long long* p) { sk_set_debug(p); }

int tc_init(TcWorkspace* ws, void* base, size_t bytes) {
  ws->base = base;
  ws->bytes = bytes;
  if (sk_init(base, bytes)) return -1;
  int dev = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&ws->num_sms, cudaDevAttrMultiProcessorCount, dev);
  return 0;
}

void tc_destroy(TcWorkspace*) {}

int gemm_tc(TcWorkspace* ws, const GemmArgs& a, cudaStream_t s) { return gemm_sk(ws->base, ws->num_sms, a, s); }

}  // namespace fl
