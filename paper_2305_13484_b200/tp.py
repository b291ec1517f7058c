"""Tensor-parallel plumbing: one process per GPU, torch.distributed for setup.

The data path (2 all-reduces per layer + the greedy-token max-reduce) runs
inside ``fl_step`` on the library's own NCCL communicator; torch.distributed
only carries the 128-byte NCCL unique id and, in device-clock mode, the
per-iteration duration every rank must agree on (the schedule is replicated
on every rank and must not diverge: each rank advances ``now`` by the max
over ranks of the measured step time).

The reference models all of this as ``TPConfig`` + ``comm_time``
(cost.py:26-33, 73-86): "two all-reduces plus one all-gather" per iteration.
"""

from __future__ import annotations

import ctypes as C

import torch
import torch.distributed as dist

from . import _lib


def make_comm_id(rank: int, src: int = 0, device=None, id_fn=None) -> bytes:
    """Rank ``src`` creates the NCCL unique id; every rank receives it."""
    if device is None:
        device = torch.device("cuda", torch.cuda.current_device()) if torch.cuda.is_available() \
            else torch.device("cpu")
    buf = torch.zeros(128, dtype=torch.uint8, device=device)
    if rank == src:
        if id_fn is None:
            raw = C.create_string_buffer(128)
            _lib.check(_lib.load().fl_comm_unique_id(raw))
            data = raw.raw[:128]
        else:
            data = id_fn()
        buf.copy_(torch.frombuffer(bytearray(data), dtype=torch.uint8))
    dist.broadcast(buf, src)
    return bytes(buf.cpu().tolist())


def max_reduce_clock(local_rank: int | None = None, device=None):
    """Returns ms -> max over ranks of ms (all ranks advance the same clock)."""
    if device is None:
        device = torch.device("cuda", local_rank) if local_rank is not None else torch.device("cpu")
    cell = torch.zeros(1, dtype=torch.float64, device=device)

    def reduce(ms: float) -> float:
        cell.fill_(ms)
        dist.all_reduce(cell, op=dist.ReduceOp.MAX)
        return float(cell.item())

    return reduce
