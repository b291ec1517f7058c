// K10: memory-shuffle compaction -- the device image of apply_shuffle
// (reference buffer.py:261-278) executing the move list of plan_shuffle
// (buffer.py:226-258).  For every move (src, dst, ctx) the live prefix
// [0, ctx) of each (layer, K/V, head) block [S, hd] is copied from physical
// slot src to dst.  One launch per shuffle boundary; source and destination
// slots are disjoint (plan pairs occupied-outside with holes-inside), so the
// copies are hazard-free.  Per-request state (next token, position,
// generation count, token history) lives in rid-indexed arrays, so nothing
// else has to move: the only bytes touched are the live KV bytes.
//
// Pure HBM stream: grid = moves x layers x 2 x heads CTAs, each copying one
// contiguous ctx*hd run with 16-byte non-allocating loads, 4 in flight/thread.
#include "common.cuh"
#include "kernels.cuh"

namespace fl {

__global__ void __launch_bounds__(256) k_shuffle(const int32_t* __restrict__ moves, int units_per_move,
                                                 uint8_t* __restrict__ kv, size_t slot_stride_b,
                                                 size_t layer_stride_b, size_t block_stride_b,
                                                 int blocks_per_slot, int row_bytes) {
  pdl_trigger();
  pdl_wait();
  const int mv = blockIdx.x / units_per_move;
  const int u = blockIdx.x % units_per_move;
  const int layer = u / blocks_per_slot, blk = u % blocks_per_slot;
  const int src = moves[3 * mv], dst = moves[3 * mv + 1], ctx = moves[3 * mv + 2];
  const size_t off = layer * layer_stride_b + blk * block_stride_b;
  const uint4* s = reinterpret_cast<const uint4*>(kv + src * slot_stride_b + off);
  uint4* d = reinterpret_cast<uint4*>(kv + dst * slot_stride_b + off);
  const int n16 = static_cast<int>((static_cast<size_t>(ctx) * row_bytes) >> 4);
  int i = threadIdx.x;
  for (; i + 3 * 256 < n16; i += 4 * 256) {
    uint4 a = ld_stream16(s + i), b = ld_stream16(s + i + 256), c = ld_stream16(s + i + 512),
          e = ld_stream16(s + i + 768);
    d[i] = a; d[i + 256] = b; d[i + 512] = c; d[i + 768] = e;
  }
  for (; i < n16; i += 256) d[i] = ld_stream16(s + i);
}

void launch_shuffle(const int32_t* moves, int n_moves, void* kv, int L, int C, int Hl, int S,
                    int hd, int dtype, cudaStream_t s) {
  if (n_moves <= 0) return;
  const size_t esz = dtype == FL_DTYPE_BF16 ? 2 : 4;
  const int row_bytes = static_cast<int>(hd * esz);
  const size_t block_b = static_cast<size_t>(S) * row_bytes;   // one (K|V, head) run
  const int blocks_per_slot = 2 * Hl;
  const size_t slot_b = block_b * blocks_per_slot;            // one slot inside a layer
  const size_t layer_b = slot_b * C;
  const int units = L * blocks_per_slot;
  launch_k(k_shuffle, dim3(n_moves * units), dim3(256), 0, s, 1, moves, units, static_cast<uint8_t*>(kv), slot_b, layer_b,
                                            block_b, blocks_per_slot, row_bytes);
}

}  // namespace fl
