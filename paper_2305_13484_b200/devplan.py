"""Device-resident shuffle planning.

`device_plan_shuffle(layout)` runs Algorithm 1 + plan_shuffle (reference
buffer.py:59-88, 226-258) as one sm_100a kernel (`fl_plan_shuffle`,
csrc/planner.cu) over the layout's window and returns the same `ShufflePlan`
the host planner builds -- bit-exact (tests/test_gpu_planner.py).  The
executor can use it to plan a shuffle boundary on the device and feed K10
straight from the device move list (`CudaExecutor(..., device_plan=True)`).
There is no CPU fallback: without the CUDA library this raises.
"""

from __future__ import annotations

import ctypes as C

from . import _lib
from .buffer import BufferLayout, ShuffleMove, ShufflePlan

MAX_WINDOW = 8192


def _torch():
    import torch
    return torch


def plan_arrays(layout: BufferLayout):
    """(occ, size) of the window slots, as the kernel consumes them."""
    win = layout.window()
    occ = [1 if s.occupant is not None else 0 for s in win]
    size = [s.size for s in win]
    return occ, size


def launch_plan(occ_d, size_d, n: int, lo: int, out_d, bytes_d, stream) -> None:
    """Stream-ordered device planning into out_d (int32 [3 + 2n]) / bytes_d (int64 [1])."""
    lib = _lib.load()
    _lib.check(lib.fl_plan_shuffle(C.c_void_p(occ_d.data_ptr()), C.c_void_p(size_d.data_ptr()), n, lo,
                                   C.c_void_p(out_d.data_ptr()), C.c_void_p(bytes_d.data_ptr()),
                                   C.c_void_p(stream)))


def device_plan_shuffle(layout: BufferLayout, device="cuda", stream=None) -> ShufflePlan:
    torch = _torch()
    occ, size = plan_arrays(layout)
    n = len(occ)
    if n > MAX_WINDOW:
        raise ValueError(f"window of {n} slots > {MAX_WINDOW}")
    s = stream if stream is not None else torch.cuda.current_stream(device)
    # inputs, kernel and read-back all ordered on one stream (the serving
    # stream is not torch's current one)
    with torch.cuda.stream(s):
        occ_d = torch.tensor(occ or [0], dtype=torch.int32, device=device)
        size_d = torch.tensor(size or [0], dtype=torch.int64, device=device)
        out_d = torch.zeros(3 + 2 * max(n, 1), dtype=torch.int32, device=device)
        bytes_d = torch.zeros(1, dtype=torch.int64, device=device)
        launch_plan(occ_d, size_d, n, layout.buffer_offset, out_d, bytes_d, s.cuda_stream)
        out = out_d.cpu().tolist()
        nbytes = int(bytes_d.item())
    offset, wlen, nm = out[0], out[1], out[2]
    slots = layout.slots
    moves = tuple(ShuffleMove(slots[out[3 + 2 * r]].occupant, out[3 + 2 * r], out[4 + 2 * r],
                              slots[out[3 + 2 * r]].size) for r in range(nm))
    return ShufflePlan(moves, offset, wlen, nbytes, layout.version)


def device_find_region(arr, device="cuda") -> int:
    """Algorithm 1 alone on a size array (nonzero = occupied), on the device."""
    lay = BufferLayout()
    for rid, v in enumerate(arr):
        lay.fuse_request(rid, v)
    for rid, v in enumerate(arr):
        if not v:
            lay.evict_request(rid)
    # keep the full array as the window (no trims): Alg. 1 sees arr itself
    return device_plan_shuffle(lay, device=device).window_offset - lay.buffer_offset
