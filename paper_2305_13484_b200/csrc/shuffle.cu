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

// Pool geometry in bytes: slot, layer and (K|V, head) block strides.
struct PoolGeom {
  uint8_t* base;
  size_t slot_b, layer_b, block_b;
};

__global__ void __launch_bounds__(256) k_shuffle(const int32_t* __restrict__ moves, int units_per_move,
                                                 PoolGeom from, PoolGeom to, int blocks_per_slot,
                                                 int row_bytes) {
  pdl_trigger();
  pdl_wait();
  const int mv = blockIdx.x / units_per_move;
  const int u = blockIdx.x % units_per_move;
  const int layer = u / blocks_per_slot, blk = u % blocks_per_slot;
  const int src = moves[3 * mv], dst = moves[3 * mv + 1], ctx = moves[3 * mv + 2];
  const uint4* s = reinterpret_cast<const uint4*>(from.base + src * from.slot_b + layer * from.layer_b +
                                                  blk * from.block_b);
  uint4* d = reinterpret_cast<uint4*>(to.base + dst * to.slot_b + layer * to.layer_b + blk * to.block_b);
  const int n16 = static_cast<int>((static_cast<size_t>(ctx) * row_bytes) >> 4);
  int i = threadIdx.x;
  for (; i + 3 * 256 < n16; i += 4 * 256) {
    uint4 a = ld_stream16(s + i), b = ld_stream16(s + i + 256), c = ld_stream16(s + i + 512),
          e = ld_stream16(s + i + 768);
    d[i] = a; d[i + 256] = b; d[i + 512] = c; d[i + 768] = e;
  }
  for (; i < n16; i += 256) d[i] = ld_stream16(s + i);
}

// K10 fed straight from the device planner's output (fl_shuffle_planned):
// plan[2] = n_moves, plan[3 + 2r] / plan[4 + 2r] = absolute logical (src,
// dst) slots; ctx[src - lo] = live positions of the source occupant.  The
// grid is sized for the worst case and strides over n_moves x units.
__global__ void __launch_bounds__(256) k_shuffle_planned(const int32_t* __restrict__ plan,
                                                         const int32_t* __restrict__ ctx_of, int lo, int C,
                                                         int units_per_move, PoolGeom pool, int blocks_per_slot,
                                                         int row_bytes) {
  pdl_trigger();
  pdl_wait();
  const int n_moves = plan[2];
  const int total = n_moves * units_per_move;
  for (int w = blockIdx.x; w < total; w += gridDim.x) {
    const int mv = w / units_per_move;
    const int u = w - mv * units_per_move;
    const int layer = u / blocks_per_slot, blk = u % blocks_per_slot;
    const int src = plan[3 + 2 * mv], dst = plan[4 + 2 * mv];
    const int ctx = ctx_of[src - lo];
    const size_t off = layer * pool.layer_b + blk * pool.block_b;
    const uint4* s = reinterpret_cast<const uint4*>(pool.base + (src % C) * pool.slot_b + off);
    uint4* d = reinterpret_cast<uint4*>(pool.base + (dst % C) * pool.slot_b + off);
    const int n16 = static_cast<int>((static_cast<size_t>(ctx) * row_bytes) >> 4);
    int i = threadIdx.x;
    for (; i + 3 * 256 < n16; i += 4 * 256) {
      uint4 a = ld_stream16(s + i), b = ld_stream16(s + i + 256), c = ld_stream16(s + i + 512),
            e = ld_stream16(s + i + 768);
      d[i] = a; d[i + 256] = b; d[i + 512] = c; d[i + 768] = e;
    }
    for (; i < n16; i += 256) d[i] = ld_stream16(s + i);
  }
}

namespace {
PoolGeom geom(void* kv, int C, int Hl, int S, size_t row_bytes) {
  PoolGeom g;
  g.base = static_cast<uint8_t*>(kv);
  g.block_b = static_cast<size_t>(S) * row_bytes;   // one (K|V, head) run [S][hd]
  g.slot_b = g.block_b * 2 * Hl;                     // one slot inside a layer
  g.layer_b = g.slot_b * C;
  return g;
}
}  // namespace

// K10 between two pools of the same model ([L][C][2][Hl][S][hd]); the
// shuffle is the case src pool == dst pool, the prefill import copies a
// staging pool (S = prompt length) into the serving pool.
void launch_kv_copy(const int32_t* moves, int n_moves, const void* src_kv, int src_C, int src_S, void* dst_kv,
                    int dst_C, int dst_S, int L, int Hl, int hd, int dtype, cudaStream_t s) {
  if (n_moves <= 0) return;
  const size_t row_bytes = hd * (dtype == FL_DTYPE_BF16 ? 2 : 4);
  const int blocks_per_slot = 2 * Hl;
  const int units = L * blocks_per_slot;
  launch_k(k_shuffle, dim3(n_moves * units), dim3(256), 0, s, 1, moves, units,
           geom(const_cast<void*>(src_kv), src_C, Hl, src_S, row_bytes), geom(dst_kv, dst_C, Hl, dst_S, row_bytes),
           blocks_per_slot, static_cast<int>(row_bytes));
}

void launch_shuffle_planned(const int32_t* plan, const int32_t* ctx_of, int lo, int max_moves, void* kv, int L,
                            int C, int Hl, int S, int hd, int dtype, cudaStream_t s) {
  if (max_moves <= 0) return;
  const size_t row_bytes = hd * (dtype == FL_DTYPE_BF16 ? 2 : 4);
  const int blocks_per_slot = 2 * Hl;
  const int units = L * blocks_per_slot;
  long long grid = static_cast<long long>(max_moves) * units;
  if (grid > 148 * 16) grid = 148 * 16;
  launch_k(k_shuffle_planned, dim3(static_cast<unsigned>(grid)), dim3(256), 0, s, 1, plan, ctx_of, lo, C, units,
           geom(kv, C, Hl, S, row_bytes), blocks_per_slot, static_cast<int>(row_bytes));
}

void launch_shuffle(const int32_t* moves, int n_moves, void* kv, int L, int C, int Hl, int S,
                    int hd, int dtype, cudaStream_t s) {
  launch_kv_copy(moves, n_moves, kv, C, S, kv, C, S, L, Hl, hd, dtype, s);
}

}  // namespace fl
