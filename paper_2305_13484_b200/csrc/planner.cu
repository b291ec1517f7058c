// Device-resident shuffle planner: Algorithm 1 (find_shuffled_memory_region,
// reference buffer.py:59-88 / PAPER.md:267-299) and plan_shuffle
// (buffer.py:226-258) for one window of the fused buffer, so a shuffle
// boundary can be planned and executed (K10) without a host round trip
// (SURVEY.md section 8f item 3).  Integer work, bit-exact with the host planner:
//
//   arr[i]   = size of window slot i if occupied, else 0     (size_array)
//   k        = #nonzero entries of arr
//   offset   = earliest o maximising sum(arr[o, o+k))        (strict improvement)
//   window   = [offset, offset + #occupants)
//   moves    = occupied slots outside the window (ascending) paired with the
//              holes inside it (ascending); bytes = sum of moved sizes
//
// One CTA of 1024 threads; the window (<= 8192 slots) lives in shared memory;
// every step is a block reduction or a segmented block scan.
#include "common.cuh"

namespace fl {

namespace {

constexpr int PL_THREADS = 1024;
constexpr int PL_MAX_N = 8192;

// inclusive scan of v[0, n) (shared memory) in place; each thread scans one
// contiguous segment serially, then the 1024 segment totals are scanned
template <typename T>
__device__ void block_scan_inclusive(T* v, int n, T* seg) {
  const int per = (n + PL_THREADS - 1) / PL_THREADS;
  const int b = threadIdx.x * per, e = min(n, b + per);
  T run = 0;
  for (int i = b; i < e; ++i) { run += v[i]; v[i] = run; }
  seg[threadIdx.x] = run;
  __syncthreads();
  // Hillis-Steele over the segment totals
  for (int off = 1; off < PL_THREADS; off <<= 1) {
    const T add = threadIdx.x >= off ? seg[threadIdx.x - off] : 0;
    __syncthreads();
    seg[threadIdx.x] += add;
    __syncthreads();
  }
  const T base = threadIdx.x ? seg[threadIdx.x - 1] : 0;
  for (int i = b; i < e; ++i) v[i] += base;
  __syncthreads();
}

__global__ void __launch_bounds__(PL_THREADS) k_plan_shuffle(const int32_t* __restrict__ occ,
                                                            const int64_t* __restrict__ size, int n,
                                                            int lo, int32_t* __restrict__ out,
                                                            long long* __restrict__ bytes) {
  extern __shared__ __align__(16) unsigned char pl_smem[];
  long long* P = reinterpret_cast<long long*>(pl_smem);                // [n + 1] prefix of arr
  int* cnt_out = reinterpret_cast<int*>(P + n + 1);                    // [n] scan of "occupied outside"
  int* cnt_hole = cnt_out + n;                                         // [n] scan of "hole inside"
  __shared__ long long seg64[PL_THREADS];
  __shared__ int seg32[PL_THREADS];
  __shared__ long long best_v[32];
  __shared__ int best_i[32];
  __shared__ int s_k, s_occ;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  if (tid == 0) { s_k = 0; s_occ = 0; P[0] = 0; }
  __syncthreads();
  int k_local = 0, occ_local = 0;
  for (int i = tid; i < n; i += PL_THREADS) {
    const long long a = occ[i] ? size[i] : 0;
    P[i + 1] = a;
    k_local += a != 0;
    occ_local += occ[i] != 0;
  }
  for (int o = 16; o; o >>= 1) {
    k_local += __shfl_xor_sync(0xffffffffu, k_local, o);
    occ_local += __shfl_xor_sync(0xffffffffu, occ_local, o);
  }
  if (lane == 0) { atomicAdd(&s_k, k_local); atomicAdd(&s_occ, occ_local); }
  __syncthreads();
  block_scan_inclusive<long long>(P + 1, n, seg64);
  const int k = s_k;
  // Alg. 1: maximise the bytes inside the length-k window; earliest wins
  long long bv = -1;
  int bi = 0x7fffffff;
  for (int o = tid; o <= n - k; o += PL_THREADS) {
    const long long inside = P[o + k] - P[o];
    if (inside > bv || (inside == bv && o < bi)) { bv = inside; bi = o; }
  }
  for (int off = 16; off; off >>= 1) {
    const long long ov = __shfl_xor_sync(0xffffffffu, bv, off);
    const int oi = __shfl_xor_sync(0xffffffffu, bi, off);
    if (ov > bv || (ov == bv && oi < bi)) { bv = ov; bi = oi; }
  }
  if (lane == 0) { best_v[warp] = bv; best_i[warp] = bi; }
  __syncthreads();
  if (warp == 0) {
    bv = best_v[lane];
    bi = best_i[lane];
    for (int off = 16; off; off >>= 1) {
      const long long ov = __shfl_xor_sync(0xffffffffu, bv, off);
      const int oi = __shfl_xor_sync(0xffffffffu, bi, off);
      if (ov > bv || (ov == bv && oi < bi)) { bv = ov; bi = oi; }
    }
    if (lane == 0) best_i[0] = k == 0 ? 0 : bi;
  }
  __syncthreads();
  const int w0 = best_i[0], w1 = w0 + s_occ;
  // plan_shuffle: occupied-outside sources and inside holes, ascending, paired
  for (int i = tid; i < n; i += PL_THREADS) {
    const bool inside = i >= w0 && i < w1;
    cnt_out[i] = (occ[i] != 0 && !inside) ? 1 : 0;
    cnt_hole[i] = (occ[i] == 0 && inside) ? 1 : 0;
  }
  __syncthreads();
  block_scan_inclusive<int>(cnt_out, n, seg32);
  block_scan_inclusive<int>(cnt_hole, n, seg32);
  const int n_src = n ? cnt_out[n - 1] : 0, n_dst = n ? cnt_hole[n - 1] : 0;
  const int n_moves = min(n_src, n_dst);
  long long moved = 0;
  for (int i = tid; i < n; i += PL_THREADS) {
    const int rs = cnt_out[i] - (i ? cnt_out[i - 1] : 0) ? cnt_out[i] - 1 : -1;   // rank if a source
    const int rd = cnt_hole[i] - (i ? cnt_hole[i - 1] : 0) ? cnt_hole[i] - 1 : -1;  // rank if a hole
    if (rs >= 0 && rs < n_moves) {
      out[3 + 2 * rs] = lo + i;
      moved += size[i];
    }
    if (rd >= 0 && rd < n_moves) out[4 + 2 * rd] = lo + i;
  }
  for (int off = 16; off; off >>= 1) moved += __shfl_xor_sync(0xffffffffu, moved, off);
  if (lane == 0) seg64[warp] = moved;
  __syncthreads();
  if (tid == 0) {
    long long tot = 0;
    for (int w = 0; w < PL_THREADS / 32; ++w) tot += seg64[w];
    out[0] = lo + w0;
    out[1] = s_occ;
    out[2] = n_moves;
    *bytes = tot;
  }
}

}  // namespace

size_t plan_smem_bytes(int n) { return static_cast<size_t>(n + 1) * 8 + static_cast<size_t>(n) * 8 + 16; }

int launch_plan_shuffle(const int32_t* occ, const int64_t* size, int n, int lo, int32_t* out,
                        long long* bytes, cudaStream_t s) {
  if (n < 0 || n > PL_MAX_N) return -1;
  static bool configured = false;
  if (!configured) {
    cudaFuncSetAttribute(k_plan_shuffle, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         static_cast<int>(plan_smem_bytes(PL_MAX_N)));
    configured = true;
  }
  k_plan_shuffle<<<1, PL_THREADS, plan_smem_bytes(n), s>>>(occ, size, n, lo, out, bytes);
  return cudaGetLastError() == cudaSuccess ? 0 : -1;
}

}  // namespace fl
