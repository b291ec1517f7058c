// K3/K5/K6/K7/K8 projections on the 5th-generation tensor cores.
//
// Decode GEMMs are skinny: M = rows of the fused window (1..512), N = weight
// rows (768..50400), K = 256..24576.  Swap-AB puts the WEIGHT tile on the
// 128-lane UMMA M side and the tokens on the UMMA N side (16..256 columns of
// TMEM), so one tcgen05.mma.cta_group::1.kind::f16 (M=128, N=BN, K=16) consumes
// a 128x16 weight slab per issue regardless of how few rows are fused.
//
//   warp 0  : TMA producer  -- cp.async.bulk.tensor 2D, SWIZZLE_128B, into a
//             STAGES-deep ring of {W 128x64, X BNx64} bf16 tiles (mbarrier tx)
//   warp 1  : TMEM allocator + single-thread MMA issuer (tcgen05.mma,
//             tcgen05.commit -> empty[stage] / done)
//   warps 2-5: epilogue -- tcgen05.ld 32x32b.x16 from TMEM (warp w%4 owns lanes
//             32(w%4)..+32), bias / GELU / residual-accumulate, coalesced stores.
//
// Split-K over grid.z fills all 148 SMs when N/128 tiles are few; partial
// tiles go to an fp32 workspace and the last-arriving CTA of a tile (counter
// in global memory, self-resetting) reduces them and runs the epilogue.
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

constexpr int TC_BM = 128;     // weight rows per tile (UMMA M)
constexpr int TC_BK = 64;      // K per stage: one 128-byte swizzle row of bf16
constexpr int TC_THREADS = 192;
constexpr int A_BYTES = TC_BM * TC_BK * 2;   // 16 KB

thread_local std::string g_tc_err;

FL_DEV uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

FL_DEV void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}

FL_DEV void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
               "r"(bytes)
               : "memory");
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

FL_DEV void tma_load_2d(const CUtensorMap* map, uint64_t* bar, void* dst, int c0, int c1) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, "
      "%4}], [%2];" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(smem_u32(bar)), "r"(c0), "r"(c1)
      : "memory");
}

// Multicast variant: the box lands at the same smem offset in every CTA of
// cta_mask and completes tx bytes on each receiver's mbarrier at that offset.
FL_DEV void tma_load_2d_mc(const CUtensorMap* map, uint64_t* bar, void* dst, int c0, int c1,
                           uint16_t cta_mask) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes.multicast::cluster"
      " [%0], [%1, {%3, %4}], [%2], %5;" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(smem_u32(bar)), "r"(c0), "r"(c1), "h"(cta_mask)
      : "memory");
}

// 2-SM (cta_group::2) load: lands in this CTA's smem, completes tx bytes on
// the LEADER CTA's mbarrier (peer bit of the shared::cluster address cleared)
FL_DEV void tma_load_2d_pair(const CUtensorMap* map, uint64_t* bar, void* dst, int c0, int c1) {
  const uint32_t leader_bar = smem_u32(bar) & 0xFEFFFFFFu;
  asm volatile(
      "cp.async.bulk.tensor.2d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, "
      "{%3, %4}], [%2];" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(leader_bar), "r"(c0), "r"(c1)
      : "memory");
}

FL_DEV void mma_bf16_pair(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc, uint32_t idesc, uint32_t acc) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem_d),
      "l"(adesc), "l"(bdesc), "r"(idesc), "r"(acc));
}

FL_DEV void mma_commit_pair(uint64_t* bar, uint16_t cta_mask) {
  asm volatile(
      "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], "
      "%1;" ::"r"(smem_u32(bar)), "h"(cta_mask)
      : "memory");
}

FL_DEV void tc_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
FL_DEV void tc_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }

// K-major operand tile [rows][64 bf16] written by TMA with 128-byte swizzle:
// 8-row (1024-byte) swizzle atoms stacked along rows -> SBO = 1024 B.
FL_DEV uint64_t smem_desc_sw128(const void* tile) {
  const uint64_t addr = smem_u32(tile);
  uint64_t d = (addr >> 4) & 0x3FFFull;    // start address
  d |= 1ull << 16;                          // LBO (unused for swizzled K-major)
  d |= (1024ull >> 4) << 32;                // SBO
  d |= 1ull << 46;                          // descriptor version (sm_100)
  d |= 2ull << 61;                          // SWIZZLE_128B
  return d;
}

// kind::f16 instruction descriptor: BF16 x BF16 -> F32, both K-major.
__host__ __device__ constexpr uint32_t instr_desc_bf16(int m, int n) {
  return (1u << 4)            // D format F32
         | (1u << 7)          // A format BF16
         | (1u << 10)         // B format BF16
         | (uint32_t(n >> 3) << 17) | (uint32_t(m >> 4) << 24);
}

FL_DEV void mma_bf16(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc, uint32_t idesc, uint32_t acc) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem_d),
      "l"(adesc), "l"(bdesc), "r"(idesc), "r"(acc));
}

FL_DEV void mma_commit(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                   smem_u32(bar))
               : "memory");
}

// commit to the same mbarrier in every CTA of cta_mask
FL_DEV void mma_commit_mc(uint64_t* bar, uint16_t cta_mask) {
  asm volatile(
      "tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], "
      "%1;" ::"r"(smem_u32(bar)), "h"(cta_mask)
      : "memory");
}

FL_DEV void tmem_ld16(uint32_t taddr, float* v) {
  uint32_t r[16];
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15},"
      " [%16];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),
        "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]),
        "=r"(r[14]), "=r"(r[15])
      : "r"(taddr));
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
  for (int i = 0; i < 16; ++i) v[i] = __uint_as_float(r[i]);
}

// 32 consecutive accumulator columns of this thread's TMEM lane; no wait --
// the caller issues several and then one tcgen05.wait::ld
FL_DEV void tmem_ld32_nowait(uint32_t taddr, uint32_t* r) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
      "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),
        "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]),
        "=r"(r[14]), "=r"(r[15]), "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]),
        "=r"(r[21]), "=r"(r[22]), "=r"(r[23]), "=r"(r[24]), "=r"(r[25]), "=r"(r[26]), "=r"(r[27]),
        "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
      : "r"(taddr));
}

template <int BN>
struct TmemCols {
  static constexpr int v = BN <= 32 ? 32 : BN <= 64 ? 64 : BN <= 128 ? 128 : 256;
};

FL_DEV uint32_t cluster_rank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}

FL_DEV void cluster_sync_all() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::
                   : "memory");
}

FL_DEV float4 ld_dsmem_f4(uint32_t local_addr, uint32_t peer) {
  uint32_t remote;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(remote) : "r"(local_addr), "r"(peer));
  float4 v;
  asm volatile("ld.shared::cluster.v4.f32 {%0,%1,%2,%3}, [%4];"
               : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w)
               : "r"(remote));
  return v;
}

// Epilogue element-wise op on 4 consecutive weight rows n..n+3 of token m.
FL_DEV void store4(void* out, size_t o, int nvalid, const float* v, int epi) {
  if (epi == EPI_STORE || epi == EPI_GELU) {
    bf16* p = static_cast<bf16*>(out) + o;
    float w[4];
#pragma unroll
    for (int j = 0; j < 4; ++j) w[j] = epi == EPI_GELU ? gelu_tanh(v[j]) : v[j];
    if (nvalid == 4 && (o & 3) == 0) {
      __nv_bfloat162 a = __floats2bfloat162_rn(w[0], w[1]), b = __floats2bfloat162_rn(w[2], w[3]);
      uint2 raw = make_uint2(*reinterpret_cast<uint32_t*>(&a), *reinterpret_cast<uint32_t*>(&b));
      *reinterpret_cast<uint2*>(p) = raw;
    } else {
      for (int j = 0; j < nvalid; ++j) p[j] = __float2bfloat16_rn(w[j]);
    }
  } else {
    float* p = static_cast<float*>(out) + o;
    if (nvalid == 4 && (o & 3) == 0) {
      float4 r = make_float4(v[0], v[1], v[2], v[3]);
      if (epi == EPI_ACC_F32) {
        const float4 x = *reinterpret_cast<float4*>(p);
        r.x += x.x; r.y += x.y; r.z += x.z; r.w += x.w;
      }
      *reinterpret_cast<float4*>(p) = r;
    } else {
      for (int j = 0; j < nvalid; ++j) p[j] = epi == EPI_ACC_F32 ? p[j] + v[j] : v[j];
    }
  }
}

// One launch = grid (ceil(N/(128*WT)), ceil(M/(MT*bn)), S), cluster (CM, 1, S).
//
// A CTA owns WT weight tiles of 128 rows and MT token sub-tiles of bn columns
// (accumulator (w, j) at TMEM column (w*MT + j)*bn, WT*MT*bn <= 512), so with
// MT covering the whole fused window every weight byte is read once per GEMM.
// The shared-memory ring is carved at run time: as many stages of
// (WT*16 KB + MT*bn*128 B) as fit (~200 KB), i.e. the deepest pipeline the
// window's width allows, one CTA per SM.  The S CTAs of a cluster split K for
// the same output tile and reduce their fp32 partials through distributed
// shared memory; S need not be a power of two (row quads are dealt out
// evenly).  The epilogue walks the accumulators in 64-column chunks:
// TMEM -> own smem [64][132] -> cluster barrier -> each CTA reduces its rows
// over the S partials -> bias / GELU / residual / argmax -> global.
constexpr int TC_MAXST = 24;

template <bool PAIR>
__global__ void __launch_bounds__(TC_THREADS, 1)
    k_gemm_tc(const __grid_constant__ CUtensorMap tma_w, const __grid_constant__ CUtensorMap tma_x,
              const bf16* __restrict__ bias, void* __restrict__ out, int M, int N, int ldo, int epi,
              int kch_total, int kch_per_split, unsigned long long* __restrict__ keys,
              int index_base, int bn, int CM, int MT, int WT, int stages, int ncols,
              int cl_split, const RopeArgs rope, unsigned long long* __restrict__ dbg) {
  // cl_split: the S K-splits form a cluster and reduce through DSMEM; otherwise
  // every split is independent and (EPI_ACC_F32) red.adds its partial.
  constexpr int RED_LD = TC_BM + 4;          // partial chunk [CH][132] fp32 (n fastest)
  constexpr int CH = 64;                     // epilogue chunk (token columns)
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  __shared__ __align__(8) uint64_t full_bar[TC_MAXST];
  __shared__ __align__(8) uint64_t empty_bar[TC_MAXST];
  __shared__ __align__(8) uint64_t done_bar;
  __shared__ uint32_t tmem_base;

  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int n_tile = blockIdx.x, split = blockIdx.z, S = gridDim.z;
  const int AB = WT * A_BYTES;
  const int XB = (CM == 2 ? bn / 2 : bn) * TC_BK * 2;   // staged token sub-tile (rows x 128 B)
  const int STAGE_BYTES = AB + MT * XB;
  const int n0 = n_tile * TC_BM * WT, m0 = blockIdx.y * MT * bn;
  const int kc0 = split * kch_per_split;
  const int nch = max(0, min(kch_per_split, kch_total - kc0));
  const uint32_t tx_bytes = CM * (AB + MT * XB);      // pair mode: the leader counts both CTAs
  const int mcount = min(MT * bn, M - m0);   // valid token columns of this tile
  const int csize = CM * (cl_split ? S : 1);
  const uint32_t crank = csize > 1 ? cluster_rank() : 0;
  const int xi = static_cast<int>(crank) % CM;          // position in the CTA pair
  const int zi = split;                                 // K split index
  const uint16_t group_mask =
      static_cast<uint16_t>(((1u << CM) - 1u) << (cl_split ? CM * zi : 0));

  // pair mode (CM == 2): the two CTAs of a cluster x-pair run one 2-SM
  // tcgen05.mma.cta_group::2 (M = 256 weight rows, each CTA holding its own 128
  // rows of A and half of the token tile B); only the leader (xi == 0) issues
  // MMAs, both CTAs' TMA loads complete on the leader's full barrier, the
  // leader's commits arrive on both CTAs' empty/done barriers.
  // (a kernel containing cta_group::2 instructions must be launched with
  // x-paired clusters, so the 1-SM and 2-SM variants are separate kernels)
  constexpr bool pair = PAIR;
  const bool leader = !pair || xi == 0;
  const int xrows = pair ? bn / 2 : bn;                 // token rows this CTA stages per sub-tile

  // ---- prologue (overlaps the predecessor kernel under PDL)
  if (threadIdx.x == 0) {
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tma_w)) : "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tma_x)) : "memory");
    for (int s = 0; s < stages; ++s) {
      mbar_init(&full_bar[s], 1);
      mbar_init(&empty_bar[s], 1);
    }
    mbar_init(&done_bar, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 1) {
    if constexpr (PAIR) {
      asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                       smem_u32(&tmem_base)),
                   "r"(ncols));
      asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;");
    } else {
      asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                       smem_u32(&tmem_base)),
                   "r"(ncols));
      asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
  }
  tc_fence_before();
  if (csize > 1) cluster_sync_all();   // peers' barriers exist before any multicast
  else __syncthreads();
  tc_fence_after();
  pdl_trigger();
  const uint32_t tmem = tmem_base;

  if (warp == 0) {
    if (lane == 0) {
      // weights do not depend on the predecessor: start streaming them first
      const int pre = min(nch, stages);
      for (int c = 0; c < pre; ++c) {
        uint8_t* a = smem + c * STAGE_BYTES;
        if (leader) mbar_expect_tx(&full_bar[c], tx_bytes);
        for (int w = 0; w < WT; ++w) {
          if constexpr (PAIR) tma_load_2d_pair(&tma_w, &full_bar[c], a + w * A_BYTES, (kc0 + c) * TC_BK, n0 + w * TC_BM);
          else tma_load_2d(&tma_w, &full_bar[c], a + w * A_BYTES, (kc0 + c) * TC_BK, n0 + w * TC_BM);
        }
      }
      pdl_wait();                                   // activations are the predecessor's output
      for (int c = 0; c < pre; ++c)
        for (int j = 0; j < MT; ++j) {
          uint8_t* dst = smem + c * STAGE_BYTES + AB + j * XB;
          if constexpr (PAIR) tma_load_2d_pair(&tma_x, &full_bar[c], dst, (kc0 + c) * TC_BK, m0 + j * bn + xi * xrows);
          else tma_load_2d(&tma_x, &full_bar[c], dst, (kc0 + c) * TC_BK, m0 + j * bn);
        }
      int s = pre % stages;
      uint32_t ph = pre / stages ? 1u : 0u;
      unsigned long long waited = 0, t_start = clock64();
      for (int c = pre; c < nch; ++c) {
        const unsigned long long tw = dbg ? clock64() : 0;
        mbar_wait(&empty_bar[s], ph ^ 1);
        if (dbg) waited += clock64() - tw;
        uint8_t* a = smem + s * STAGE_BYTES;
        if (leader) mbar_expect_tx(&full_bar[s], tx_bytes);
        const int k = (kc0 + c) * TC_BK;
        for (int w = 0; w < WT; ++w) {
          if constexpr (PAIR) tma_load_2d_pair(&tma_w, &full_bar[s], a + w * A_BYTES, k, n0 + w * TC_BM);
          else tma_load_2d(&tma_w, &full_bar[s], a + w * A_BYTES, k, n0 + w * TC_BM);
        }
        for (int j = 0; j < MT; ++j) {
          uint8_t* dst = a + AB + j * XB;
          if constexpr (PAIR) tma_load_2d_pair(&tma_x, &full_bar[s], dst, k, m0 + j * bn + xi * xrows);
          else tma_load_2d(&tma_x, &full_bar[s], dst, k, m0 + j * bn);
        }
        if (++s == stages) { s = 0; ph ^= 1; }
      }
      if (dbg) {
        const int b = blockIdx.x + gridDim.x * (blockIdx.y + gridDim.y * blockIdx.z);
        dbg[4 * b + 0] = waited;
        dbg[4 * b + 1] = clock64() - t_start;
      }
    }
  } else if (warp == 1) {
    if (lane == 0 && leader) {
      const uint32_t idesc = instr_desc_bf16(pair ? 2 * TC_BM : TC_BM, bn);
      int s = 0;
      uint32_t ph = 0;
      unsigned long long waited = 0, t_start = clock64();
      for (int c = 0; c < nch; ++c) {
        const unsigned long long tw = dbg ? clock64() : 0;
        mbar_wait(&full_bar[s], ph);
        if (dbg) waited += clock64() - tw;
        tc_fence_after();
        const uint8_t* a = smem + s * STAGE_BYTES;
        for (int w = 0; w < WT; ++w) {
          const uint64_t ad = smem_desc_sw128(a + w * A_BYTES);
          for (int j = 0; j < MT; ++j) {
            const uint64_t bd = smem_desc_sw128(a + AB + j * XB);
#pragma unroll
            for (int k = 0; k < TC_BK / 16; ++k) {   // 16 bf16 = 32 bytes = 2 descriptor units
              if constexpr (PAIR)
                mma_bf16_pair(tmem + (w * MT + j) * bn, ad + 2 * k, bd + 2 * k, idesc, (c | k) != 0);
              else
                mma_bf16(tmem + (w * MT + j) * bn, ad + 2 * k, bd + 2 * k, idesc, (c | k) != 0);
            }
          }
        }
        if constexpr (PAIR) mma_commit_pair(&empty_bar[s], group_mask);
        else mma_commit(&empty_bar[s]);
        if (++s == stages) { s = 0; ph ^= 1; }
      }
      if constexpr (PAIR) mma_commit_pair(&done_bar, group_mask);
      else mma_commit(&done_bar);
      if (dbg) {
        const int b = blockIdx.x + gridDim.x * (blockIdx.y + gridDim.y * blockIdx.z);
        dbg[4 * b + 2] = waited;
        dbg[4 * b + 3] = clock64() - t_start;
      }
    }
  } else {
    pdl_wait();     // EPI_ACC_F32 reads `out`, written by predecessors
    if (nch > 0) {
      mbar_wait(&done_bar, 0);
      tc_fence_after();
    }
  }
  __syncwarp();

  // ---- epilogue, direct path (no split-K): each epilogue thread owns one
  // weight row (its TMEM lane) and streams its accumulator row out 32 token
  // columns at a time -- per store instruction a warp writes 32 consecutive
  // weight rows of one token (a coalesced 64/128-byte segment).
  if (!cl_split) {
    if (warp >= 2) {
      const int quarter = warp & 3;
      const int row = quarter * 32 + lane;
      for (int w = 0; w < WT; ++w) {
        const int n = n0 + w * TC_BM + row;
        const bool nok = n < N;
        const float bv = (bias && nok && split == 0) ? __bfloat162float(bias[n]) : 0.f;
        for (int cb = 0; cb < mcount; cb += 32) {
          uint32_t r[32];
          if (nch > 0) {
            tmem_ld32_nowait(tmem + (static_cast<uint32_t>(quarter * 32) << 16) + w * MT * bn + cb, r);
            asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
          } else {
#pragma unroll
            for (int j = 0; j < 32; ++j) r[j] = 0u;
          }
          const int ncol = min(32, mcount - cb);
          if (epi == EPI_QKV) {
            // q/k/v section, head and dim of this weight row; rotary partner is a
            // lane of this warp (GPT-J: n^1; NeoX: n +- rot/2 inside the head's
            // first rot dims -- a head starts on a 32-row boundary for hd % 32 == 0)
            const int D = rope.Hl * rope.hd;
            const int sec = n / D, rem = n - sec * D;
            const int hh = rem / rope.hd, ii = rem - hh * rope.hd;
            const bool rot_row = sec < 2 && ii < rope.rot;
            int src = lane, jf = 0;
            float sgn = 0.f;
            if (rope.family == FL_FAMILY_GPTJ) {
              src = lane ^ 1; jf = ii >> 1; sgn = (ii & 1) ? 1.f : -1.f;
            } else if (rope.family == FL_FAMILY_NEOX) {
              const int half = rope.rot >> 1;
              src = ii < half ? lane + half : lane - half;
              jf = ii < half ? ii : ii - half;
              sgn = ii < half ? -1.f : 1.f;
            }
            src = rot_row ? src : lane;
            const float inv_freq = exp2f(-(2.f * jf / max(rope.rot, 1)) * 13.287712379549449f);
#pragma unroll 4
            for (int j = 0; j < 32; ++j) {
              if (j >= ncol) break;
              float x = __uint_as_float(r[j]) + bv;
              const float xp = __shfl_sync(0xffffffffu, x, src);
              const int mg = m0 + cb + j;
              const int pos = rope.row_pos[mg];
              if (rot_row) {
                float sn, cs;
                sincosf(static_cast<float>(pos) * inv_freq, &sn, &cs);
                x = x * cs + sgn * xp * sn;
              }
              if (!nok) continue;
              if (sec == 0) {
                static_cast<bf16*>(rope.q_out)[static_cast<size_t>(mg) * D + rem] = __float2bfloat16_rn(x);
              } else if (rope.rows[mg].kind != FL_ROW_ORPHAN) {
                const size_t slot = rope.rows[mg].slot;
                const size_t o = (((slot * 2 + (sec - 1)) * rope.Hl + hh) * rope.S + pos) * rope.hd + ii;
                static_cast<bf16*>(rope.kv_layer)[o] = __float2bfloat16_rn(x);
              }
            }
          } else if (epi == EPI_ARGMAX) {
#pragma unroll 4
            for (int j = 0; j < 32; ++j) {
              if (j >= ncol) break;
              unsigned long long key = nok ? argmax_key(__uint_as_float(r[j]) + bv, index_base + n) : 0ull;
#pragma unroll
              for (int o = 1; o < 32; o <<= 1) {
                const unsigned long long other = __shfl_xor_sync(0xffffffffu, key, o);
                key = other > key ? other : key;
              }
              if (lane == 0 && key) atomicMax(&keys[m0 + cb + j], key);
            }
          } else if (nok) {
#pragma unroll 8
            for (int j = 0; j < 32; ++j) {
              if (j >= ncol) break;
              const float x = __uint_as_float(r[j]) + bv;
              const size_t o = static_cast<size_t>(m0 + cb + j) * ldo + n;
              switch (epi) {
                case EPI_STORE: static_cast<bf16*>(out)[o] = __float2bfloat16_rn(x); break;
                case EPI_GELU: static_cast<bf16*>(out)[o] = __float2bfloat16_rn(gelu_tanh(x)); break;
                case EPI_ACC_F32:
                  if (S > 1) atomicAdd(static_cast<float*>(out) + o, x);   // red.global.add
                  else static_cast<float*>(out)[o] += x;
                  break;
                default: static_cast<float*>(out)[o] = x; break;
              }
            }
          }
        }
      }
    }
    tc_fence_before();
    __syncwarp();
    if (csize > 1) cluster_sync_all();   // the pair's TMEM is freed jointly
    else __syncthreads();
    if (warp == 1) {
      tc_fence_after();
      if constexpr (PAIR)
        asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(ncols));
      else
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(ncols));
    }
    return;
  }

  // ---- epilogue, one 64-column chunk at a time (all 192 threads keep the
  // cluster barriers in lock step; warps 2..5 move the data).  This CTA
  // reduces row quads [q_lo, q_hi) of each 128-row weight tile.
  const int q_lo = zi * 32 / S, q_hi = (zi + 1) * 32 / S;
  const int nq = q_hi - q_lo;
  float* red = reinterpret_cast<float*>(smem);
  const uint32_t red_base = smem_u32(smem);
  const int quarter = warp & 3;
  const int row = quarter * 32 + lane;
  const int nchunk = (mcount + CH - 1) / CH;
  for (int it = 0; it < WT * nchunk; ++it) {
    const int w = it / nchunk;                   // weight tile
    const int cb = (it % nchunk) * CH;           // first token column of the chunk
    const int ncol = min(CH, mcount - cb);
    const int nw0 = n0 + w * TC_BM;
    if (warp >= 2) {
      if (nch > 0) {
        const uint32_t taddr = tmem + (static_cast<uint32_t>(quarter * 32) << 16) + w * MT * bn + cb;
        for (int c0 = 0; c0 < ncol; c0 += 16) {
          float v[16];
          tmem_ld16(taddr + c0, v);
#pragma unroll
          for (int j = 0; j < 16; ++j) red[(c0 + j) * RED_LD + row] = v[j];
        }
      } else {
        for (int c0 = 0; c0 < ncol; ++c0) red[c0 * RED_LD + row] = 0.f;
      }
    }
    tc_fence_before();
    if (csize > 1) cluster_sync_all();
    else __syncthreads();
    if (warp >= 2) {
      const int total = nq * ncol;
      for (int base = 0; base < total; base += 128) {
        const int e = base + threadIdx.x - 64;
        const bool valid = e < total;
        const int m = valid ? e / nq : 0;
        const int r0 = (q_lo + (valid ? e % nq : 0)) * 4;
        const uint32_t off = static_cast<uint32_t>((m * RED_LD + r0) * 4);
        float acc[4] = {0.f, 0.f, 0.f, 0.f};
        if (valid) {
          float4 t[8];
#pragma unroll
          for (int p = 0; p < 8; ++p)      // all peer loads in flight at once
            if (p < S)
              t[p] = S > 1 ? ld_dsmem_f4(red_base + off, static_cast<uint32_t>(xi + CM * p))
                           : *reinterpret_cast<const float4*>(smem + off);
#pragma unroll
          for (int p = 0; p < 8; ++p)
            if (p < S) {
              acc[0] += t[p].x; acc[1] += t[p].y; acc[2] += t[p].z; acc[3] += t[p].w;
            }
        }
        const int n = nw0 + r0;
        const int nvalid = valid ? max(0, min(4, N - n)) : 0;
        if (bias) {
#pragma unroll
          for (int j = 0; j < 4; ++j) acc[j] += j < nvalid ? __bfloat162float(bias[n + j]) : 0.f;
        }
        const int mg = m0 + cb + m;
        if (epi == EPI_ARGMAX) {
          // greedy token: max logit, lowest index; S == 1 here, so the 32
          // lanes of a warp hold one token's 128 weight rows: warp-reduce,
          // then one 64-bit atomicMax per (token, CTA)
          unsigned long long key = 0ull;
#pragma unroll
          for (int j = 0; j < 4; ++j)
            if (j < nvalid) {
              const unsigned long long k2 = argmax_key(acc[j], index_base + n + j);
              key = k2 > key ? k2 : key;
            }
#pragma unroll
          for (int o = 1; o < 32; o <<= 1) {
            const unsigned long long other = __shfl_xor_sync(0xffffffffu, key, o);
            key = other > key ? other : key;
          }
          if (valid && lane == 0 && key) atomicMax(&keys[mg], key);
        } else if (nvalid > 0) {
          store4(out, static_cast<size_t>(mg) * ldo + n, nvalid, acc, epi);
        }
      }
    }
    // the chunk buffer is rewritten next round; peers may still read it
    __syncwarp();
    if (csize > 1) cluster_sync_all();
    else __syncthreads();
  }
  if (warp == 1) {
    tc_fence_after();
    if constexpr (PAIR)
      asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(ncols));
    else
      asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(ncols));
  }
}

// ------------------------------------------------------------------ host side
PFN_cuTensorMapEncodeTiled_v12000 g_encode = nullptr;

struct MapKey {
  const void* ptr;
  uint64_t rows, cols, ld;
  uint32_t box_rows;
  bool operator<(const MapKey& o) const {
    return std::tie(ptr, rows, cols, ld, box_rows) < std::tie(o.ptr, o.rows, o.cols, o.ld, o.box_rows);
  }
};

using MapCache = std::map<MapKey, CUtensorMap>;

bool make_map(MapCache& cache, const void* ptr, uint64_t rows, uint64_t cols, uint64_t ld,
              uint32_t box_rows, CUtensorMap** out) {
  MapKey key{ptr, rows, cols, ld, box_rows};
  auto it = cache.find(key);
  if (it != cache.end()) {
    *out = &it->second;
    return true;
  }
  CUtensorMap map;
  cuuint64_t dims[2] = {cols, rows};
  cuuint64_t strides[1] = {ld * 2};
  cuuint32_t box[2] = {TC_BK, box_rows};
  cuuint32_t estr[2] = {1, 1};
  CUresult r = g_encode(&map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(ptr), dims,
                        strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                        CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                        CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) {
    char buf[160];
    snprintf(buf, sizeof buf, "cuTensorMapEncodeTiled failed (%d) rows=%llu cols=%llu", (int)r,
             (unsigned long long)rows, (unsigned long long)cols);
    g_tc_err = buf;
    return false;
  }
  *out = &(cache[key] = map);
  return true;
}

constexpr int TC_SMEM_BUDGET = 200 * 1024;   // stage ring (the epilogue reuses it)
unsigned long long* g_dbg = nullptr;          // pipeline wait counters (diagnostics)

int launch_tc(const GemmArgs& a, const CUtensorMap* mw, const CUtensorMap* mx, int splits, int kpc,
              int bn, int cm, int mt, int wt, cudaStream_t s) {
  // K splits of a residual-accumulating GEMM red.add straight into the fp32
  // residual (no cluster); other epilogues reduce through DSMEM in a cluster
  const int cl_split = (splits > 1 && a.epi != EPI_ACC_F32) ? 1 : 0;
  static bool configured = false;
  if (!configured) {
    for (auto k : {k_gemm_tc<false>, k_gemm_tc<true>}) {
      cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, TC_SMEM_BUDGET + 1024);
      cudaFuncSetAttribute(k, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    }
    configured = true;
  }
  const int stage_bytes = wt * A_BYTES + mt * (bn / cm) * TC_BK * 2;
  int stages = TC_SMEM_BUDGET / stage_bytes;
  if (stages > TC_MAXST) stages = TC_MAXST;
  if (stages < 2) {
    g_tc_err = "token tile too wide for the stage ring";
    return -1;
  }
  const int cols = wt * mt * bn;
  const int ncols = cols <= 32 ? 32 : cols <= 64 ? 64 : cols <= 128 ? 128 : cols <= 256 ? 256 : 512;
  dim3 grid((a.N + wt * TC_BM - 1) / (wt * TC_BM), (a.M + mt * bn - 1) / (mt * bn), splits);
  const int smem = stages * stage_bytes + 1024;
  cudaError_t e = launch_k(cm == 2 ? k_gemm_tc<true> : k_gemm_tc<false>, grid, dim3(TC_THREADS), smem, s, dim3(cm, 1, cl_split ? splits : 1), *mw, *mx,
                           static_cast<const bf16*>(a.bias), a.out, a.M, a.N, a.ldo, a.epi,
                           a.K / TC_BK, kpc, a.keys, a.index_base, bn, cm, mt, wt, stages, ncols,
                           cl_split, a.rope, g_dbg);
  if (e != cudaSuccess) {
    char buf[256];
    snprintf(buf, sizeof buf, "k_gemm_tc launch (grid %u,%u,%u cluster %d,1,%d smem %d stages %d bn %d): %s",
             grid.x, grid.y, grid.z, cm, splits, smem, stages, bn, cudaGetErrorString(e));
    g_tc_err = buf;
    return -1;
  }
  return 0;
}

}  // namespace

size_t tc_workspace_bytes(int, int) { return sk_workspace_bytes(); }

const char* tc_last_error() { return g_tc_err.empty() ? sk_last_error() : g_tc_err.c_str(); }
void tc_set_debug(unsigned long long* p) { g_dbg = p; sk_set_debug(p); }

int tc_init(TcWorkspace* ws, void* base, size_t bytes) {
  if (!g_encode) {
    cudaDriverEntryPointQueryResult q;
    void* fn = nullptr;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q) != cudaSuccess ||
        !fn) {
      g_tc_err = "cuTensorMapEncodeTiled entry point unavailable";
      return -1;
    }
    g_encode = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fn);
  }
  ws->base = base;
  ws->bytes = bytes;
  if (sk_init(base, bytes)) {
    g_tc_err = sk_last_error();
    return -1;
  }
  int dev = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&ws->num_sms, cudaDevAttrMultiProcessorCount, dev);
  if (!ws->maps) ws->maps = new MapCache();
  return 0;
}

void tc_destroy(TcWorkspace* ws) {
  delete static_cast<MapCache*>(ws->maps);
  ws->maps = nullptr;
}

int gemm_tc(TcWorkspace* ws, const GemmArgs& a, cudaStream_t s) {
  if (a.M <= 0 || a.N <= 0) return 0;
  if (a.dtype != FL_DTYPE_BF16 || a.K % TC_BK || a.ldx % 8) {
    g_tc_err = "tensor-core GEMM needs bf16, K % 64 == 0 and 16-byte aligned rows";
    return -1;
  }
  // default: the persistent stream-K pair kernel (gemm_sk.cu); FL_GEMM_LEGACY=1
  // selects the per-tile cluster-split kernel below (kept for comparison)
  static const bool legacy = getenv("FL_GEMM_LEGACY") != nullptr;
  if (!legacy) return gemm_sk(ws->base, ws->num_sms, a, s);
  if (a.w_tiled || a.nsplit) {
    g_tc_err = "tiled weights and dual GEMMs need the stream-K GEMM (unset FL_GEMM_LEGACY)";
    return -1;
  }
  MapCache& cache = *static_cast<MapCache*>(ws->maps);
  // Token tiling: the whole window in one CTA when it fits TMEM (MT sub-tiles
  // of <= 256 columns, MT*bn <= 512), so each weight byte is read once.
  static const int force_mt = getenv("FL_TC_MT") ? atoi(getenv("FL_TC_MT")) : 0;
  static const int force_wt = getenv("FL_TC_WT") ? atoi(getenv("FL_TC_WT")) : 0;
  const int mt = force_mt ? force_mt : (a.M <= 256 ? 1 : 2);
  const int span = 256 * mt;
  const int ntiles_m = (a.M + span - 1) / span;
  const int per_cta = (a.M + ntiles_m - 1) / ntiles_m;
  const int bn = (((per_cta + mt - 1) / mt) + 15) / 16 * 16;
  const int wt = force_wt ? force_wt : 1;
  const int ntn = (a.N + wt * TC_BM - 1) / (wt * TC_BM);
  const int tiles = ntn * ntiles_m;
  const int kch = a.K / TC_BK;
  // split K across a cluster so the grid covers the SMs once (one CTA per
  // SM, deepest ring); any S in 1..8, at least 2 K chunks per split; narrow
  // token tiles stop at 4 (cluster barriers dominate tiny tiles)
  static const int force_s = getenv("FL_TC_SPLIT") ? atoi(getenv("FL_TC_SPLIT")) : 0;
  int S = 1;
  if (a.epi != EPI_ARGMAX) {
    const int smax = (bn >= 128 || a.epi == EPI_ACC_F32) ? 8 : 4;
    // (EPI_QKV is only ever requested when the caller accepts S == 1)
    while (S < smax && tiles * (S + 1) <= ws->num_sms && kch / (S + 1) >= 2) ++S;
  }
  if (force_s > 0 && a.epi != EPI_ARGMAX) S = force_s;
  // 2-SM pairs (cta_group::2, M = 256) for wide token tiles: half the token
  // bytes staged per SM and per MMA; needs an even count of 128-row tiles
  static const int force_pair = getenv("FL_TC_PAIR") ? atoi(getenv("FL_TC_PAIR")) : -1;
  const bool cl_split = S > 1 && a.epi != EPI_ACC_F32;
  int cm = (bn >= 64 && ntn % 2 == 0 && wt == 1 && !cl_split) ? 2 : 1;
  if (force_pair == 0) cm = 1;
  if (force_pair == 1 && ntn % 2 == 0 && wt == 1 && !cl_split) cm = 2;
  const int kpc2 = (kch + S - 1) / S;
  CUtensorMap *mw, *mx;
  if (!make_map(cache, a.w, a.N, a.K, a.K, TC_BM, &mw)) return -1;
  if (!make_map(cache, a.x, a.mcap > a.M ? a.mcap : a.M, a.K, a.ldx, bn / cm, &mx)) return -1;
  // the fused QKV epilogue needs whole sums in registers: with a clustered
  // K split it falls back to a plain store (return 2: caller runs k_rope_append)
  if (a.epi == EPI_QKV && S > 1) {
    GemmArgs b = a;
    b.epi = EPI_STORE;
    return launch_tc(b, mw, mx, S, kpc2, bn, cm, mt, wt, s) ? -1 : 2;
  }
  return launch_tc(a, mw, mx, S, kpc2, bn, cm, mt, wt, s);
}

}  // namespace fl
