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

template <int BN>
struct TmemCols {
  static constexpr int v = BN <= 32 ? 32 : BN <= 64 ? 64 : BN <= 128 ? 128 : 256;
};

template <int BN, int STAGES>
__global__ void __launch_bounds__(TC_THREADS, 1)
    k_gemm_tc(const __grid_constant__ CUtensorMap tma_w, const __grid_constant__ CUtensorMap tma_x,
              const bf16* __restrict__ bias, void* __restrict__ out, int M, int N, int ldo, int epi,
              int kch_total, int kch_per_split, int* __restrict__ counters,
              float* __restrict__ partials) {
  constexpr int B_BYTES = BN * TC_BK * 2;
  constexpr int STAGE_BYTES = A_BYTES + B_BYTES;
  constexpr int NCOLS = TmemCols<BN>::v;
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  __shared__ __align__(8) uint64_t full_bar[STAGES];
  __shared__ __align__(8) uint64_t empty_bar[STAGES];
  __shared__ __align__(8) uint64_t done_bar;
  __shared__ uint32_t tmem_base;
  __shared__ int s_last;

  // 1024-byte alignment for the swizzle atoms
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int n_tile = blockIdx.x, m_tile = blockIdx.y, split = blockIdx.z, splits = gridDim.z;
  const int n0 = n_tile * TC_BM, m0 = m_tile * BN;
  const int kc0 = split * kch_per_split;
  const int nch = min(kch_per_split, kch_total - kc0);

  if (threadIdx.x == 0) {
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tma_w)) : "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tma_x)) : "memory");
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(&full_bar[s], 1);
      mbar_init(&empty_bar[s], 1);
    }
    mbar_init(&done_bar, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                     smem_u32(&tmem_base)),
                 "r"(NCOLS));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = tmem_base;

  if (warp == 0) {
    if (lane == 0) {
      for (int c = 0; c < nch; ++c) {
        const int s = c % STAGES;
        const uint32_t ph = (c / STAGES) & 1;
        mbar_wait(&empty_bar[s], ph ^ 1);
        uint8_t* a = smem + s * STAGE_BYTES;
        uint8_t* b = a + A_BYTES;
        mbar_expect_tx(&full_bar[s], STAGE_BYTES);
        const int k = (kc0 + c) * TC_BK;
        tma_load_2d(&tma_w, &full_bar[s], a, k, n0);
        tma_load_2d(&tma_x, &full_bar[s], b, k, m0);
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {
      constexpr uint32_t idesc = instr_desc_bf16(TC_BM, BN);
      for (int c = 0; c < nch; ++c) {
        const int s = c % STAGES;
        const uint32_t ph = (c / STAGES) & 1;
        mbar_wait(&full_bar[s], ph);
        tc_fence_after();
        const uint8_t* a = smem + s * STAGE_BYTES;
        const uint64_t ad = smem_desc_sw128(a);
        const uint64_t bd = smem_desc_sw128(a + A_BYTES);
#pragma unroll
        for (int k = 0; k < TC_BK / 16; ++k)   // 16 bf16 = 32 bytes = 2 descriptor units
          mma_bf16(tmem, ad + 2 * k, bd + 2 * k, idesc, (c | k) != 0);
        mma_commit(&empty_bar[s]);
      }
      mma_commit(&done_bar);
    }
  } else {
    // ---------------- epilogue (warps 2..5)
    const int quarter = warp & 3;            // TMEM lane quarter this warp may read
    const int row = quarter * 32 + lane;     // weight row within the tile
    const int n = n0 + row;
    mbar_wait(&done_bar, 0);
    tc_fence_after();
    const uint32_t taddr = tmem + (static_cast<uint32_t>(quarter * 32) << 16);
    const int mcount = min(BN, M - m0);
    const size_t tile_id = static_cast<size_t>(m_tile) * gridDim.x + n_tile;
    if (splits > 1) {
      float* part = partials + (tile_id * splits + split) * (size_t)(TC_BM * BN);
      for (int c0 = 0; c0 < BN; c0 += 16) {
        float v[16];
        tmem_ld16(taddr + c0, v);
#pragma unroll
        for (int j = 0; j < 16; ++j) part[(c0 + j) * TC_BM + row] = v[j];
      }
      __threadfence();
      asm volatile("bar.sync 1, 128;");
      if (warp == 2 && lane == 0) {
        const int prev = atomicAdd(&counters[tile_id], 1);
        s_last = (prev == splits - 1);
        if (s_last) counters[tile_id] = 0;   // self-reset for the next GEMM
      }
      asm volatile("bar.sync 1, 128;");
      if (!s_last) goto teardown;
      __threadfence();
    }
    {
      const float bv = (bias && n < N) ? __bfloat162float(bias[n]) : 0.f;
      for (int c0 = 0; c0 < BN; c0 += 16) {
        float v[16];
        if (splits > 1) {
#pragma unroll
          for (int j = 0; j < 16; ++j) v[j] = 0.f;
          const float* p0 = partials + tile_id * splits * (size_t)(TC_BM * BN);
          for (int sp = 0; sp < splits; ++sp) {
            const float* p = p0 + sp * (size_t)(TC_BM * BN);
#pragma unroll
            for (int j = 0; j < 16; ++j) v[j] += __ldcg(p + (c0 + j) * TC_BM + row);
          }
        } else {
          tmem_ld16(taddr + c0, v);
        }
        if (n < N) {
#pragma unroll
          for (int j = 0; j < 16; ++j) {
            const int m = c0 + j;
            if (m < mcount) {
              const float x = v[j] + bv;
              const size_t o = static_cast<size_t>(m0 + m) * ldo + n;
              switch (epi) {
                case EPI_STORE: static_cast<bf16*>(out)[o] = __float2bfloat16_rn(x); break;
                case EPI_GELU: static_cast<bf16*>(out)[o] = __float2bfloat16_rn(gelu_tanh(x)); break;
                case EPI_ACC_F32: static_cast<float*>(out)[o] += x; break;
                default: static_cast<float*>(out)[o] = x; break;
              }
            }
          }
        }
      }
    }
  }
teardown:
  tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(NCOLS));
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

constexpr size_t TC_COUNTERS = 4096;
constexpr size_t TC_MAX_PARTIAL_TILES = 160;   // split-K CTAs (<= SM count) writing a partial

template <int BN, int STAGES>
int launch_bn(TcWorkspace* ws, const GemmArgs& a, const CUtensorMap* mw, const CUtensorMap* mx,
              int splits, int kpc, cudaStream_t s) {
  constexpr int smem = STAGES * (A_BYTES + BN * TC_BK * 2) + 1024;
  static bool configured = false;
  if (!configured) {
    cudaFuncSetAttribute(k_gemm_tc<BN, STAGES>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    configured = true;
  }
  dim3 grid((a.N + TC_BM - 1) / TC_BM, (a.M + BN - 1) / BN, splits);
  k_gemm_tc<BN, STAGES><<<grid, TC_THREADS, smem, s>>>(
      *mw, *mx, static_cast<const bf16*>(a.bias), a.out, a.M, a.N, a.ldo, a.epi, a.K / TC_BK, kpc,
      ws->counters, ws->partials);
  return 0;
}

}  // namespace

size_t tc_workspace_bytes(int max_rows, int) {
  (void)max_rows;
  return TC_COUNTERS * sizeof(int) + TC_MAX_PARTIAL_TILES * TC_BM * 256 * sizeof(float);
}

const char* tc_last_error() { return g_tc_err.c_str(); }

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
  if (bytes < tc_workspace_bytes(0, 0)) {
    g_tc_err = "tensor-core workspace too small";
    return -1;
  }
  ws->base = base;
  ws->bytes = bytes;
  ws->counters = static_cast<int*>(base);
  ws->partials = reinterpret_cast<float*>(static_cast<char*>(base) + TC_COUNTERS * sizeof(int));
  ws->partial_floats = TC_MAX_PARTIAL_TILES * TC_BM * 256;
  int dev = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&ws->num_sms, cudaDevAttrMultiProcessorCount, dev);
  if (cudaMemset(ws->counters, 0, TC_COUNTERS * sizeof(int)) != cudaSuccess) {
    g_tc_err = "counter memset failed";
    return -1;
  }
  ws->maps = new MapCache();
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
  MapCache& cache = *static_cast<MapCache*>(ws->maps);
  const int bn = a.M <= 16 ? 16 : a.M <= 32 ? 32 : a.M <= 64 ? 64 : a.M <= 128 ? 128 : 256;
  CUtensorMap *mw, *mx;
  if (!make_map(cache, a.w, a.N, a.K, a.K, TC_BM, &mw)) return -1;
  if (!make_map(cache, a.x, a.mcap > a.M ? a.mcap : a.M, a.K, a.ldx, bn, &mx)) return -1;
  const int tiles = ((a.N + TC_BM - 1) / TC_BM) * ((a.M + bn - 1) / bn);
  const int kch = a.K / TC_BK;
  int splits = 1;
  if (tiles < ws->num_sms) {
    splits = ws->num_sms / tiles;
    if (splits > kch / 2) splits = kch / 2 > 0 ? kch / 2 : 1;
    if (splits > 16) splits = 16;
    while (splits > 1 && (size_t)tiles * splits * TC_BM * bn > ws->partial_floats) --splits;
    if ((size_t)tiles > TC_COUNTERS) splits = 1;
  }
  const int kpc = (kch + splits - 1) / splits;
  splits = (kch + kpc - 1) / kpc;
  switch (bn) {
    case 16: return launch_bn<16, 8>(ws, a, mw, mx, splits, kpc, s);
    case 32: return launch_bn<32, 8>(ws, a, mw, mx, splits, kpc, s);
    case 64: return launch_bn<64, 6>(ws, a, mw, mx, splits, kpc, s);
    case 128: return launch_bn<128, 4>(ws, a, mw, mx, splits, kpc, s);
    default: return launch_bn<256, 4>(ws, a, mw, mx, splits, kpc, s);
  }
}

}  // namespace fl
