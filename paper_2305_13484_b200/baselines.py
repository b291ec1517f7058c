"""Dynamic batching -- the comparison discipline of config C5.

Drop-in for the reference's ``run_dynamic_batching`` (baselines.py:51-127):
arrivals are grouped into fixed windows anchored at the first arrival
(``max_batch`` chunks dispatch when they fill), one instance runs the
batches FIFO, a batch dispatches when its window closes, its members are
preprocessed and the previous batch is done, and it runs as long as its
longest member with every member riding along (nothing joins or leaves
mid-batch).  With ``executor=None`` and the cost clock the trace is
identical to the reference's (tests/test_baselines_golden.py).

With a ``CudaExecutor`` each batch really runs on the B200: its members
take slots 0..B-1 of a fresh window and every iteration is one ``fl_step``
over the whole batch; members past their end marker stay in the window as
ORPHAN rows (computed and discarded -- the rigid batch keeps paying for
them, which is exactly what temporal fusion avoids).
"""

from __future__ import annotations

import math
from dataclasses import dataclass

from .buffer import BufferLayout, Slot
from .core import Request
from .cost import CostParams, TPConfig, iteration_time
from .errors import CapacityExceeded, InvalidParam
from .trace import EventKind, Trace, TraceEvent


@dataclass(frozen=True)
class BatchWindowConfig:
    window_ms: float
    max_batch: int | None = None

    def __post_init__(self):
        if self.window_ms < 0:
            raise InvalidParam("window_ms must be >= 0")
        if self.max_batch is not None and self.max_batch < 1:
            raise InvalidParam("max_batch must be >= 1 when set")


def _partition(ordered, cfg: BatchWindowConfig) -> list:
    """[(members, nominal dispatch time)] in dispatch order."""
    if cfg.window_ms == 0:
        return [([r], r.arrival_time) for r in ordered]
    t0 = ordered[0].arrival_time
    windows: dict = {}
    for r in ordered:
        windows.setdefault(math.floor((r.arrival_time - t0) / cfg.window_ms), []).append(r)
    out = []
    for idx in sorted(windows):
        close = t0 + (idx + 1) * cfg.window_ms
        chunk = []
        for r in windows[idx]:
            chunk.append(r)
            if cfg.max_batch is not None and len(chunk) == cfg.max_batch:
                out.append((chunk, r.arrival_time))
                chunk = []
        if chunk:
            out.append((chunk, close))
    return out


class _BatchStream:
    """The slice of the FusionStream surface an executor reads."""

    def __init__(self, clock: str):
        self.layout = BufferLayout()
        self.clock = clock
        self.iteration_index = 0


def run_dynamic_batching(requests, cfg: BatchWindowConfig, params: CostParams,
                         tp: TPConfig | None = None, record_tokens: bool = True, *,
                         executor=None, clock: str = "cost") -> Trace:
    if clock not in ("cost", "device"):
        raise InvalidParam(f"clock must be 'cost' or 'device', got {clock!r}")
    if clock == "device" and executor is None:
        raise InvalidParam("clock='device' needs an executor")
    from .engine import check_tp
    check_tp(tp or TPConfig(), executor, clock)
    tp = tp or TPConfig()
    ordered = sorted(requests, key=lambda r: (r.arrival_time, r.request_id))
    ev = []
    for r in ordered:
        ev.append(TraceEvent(r.arrival_time, EventKind.ARRIVED, r.request_id, None))
        ev.append(TraceEvent(r.arrival_time, EventKind.PREPROCESS_START, r.request_id, None))
        ev.append(TraceEvent(r.arrival_time + params.preprocess_ms, EventKind.PREPROCESS_DONE,
                             r.request_id, None))
    trace = Trace("dynamic_batching", ev)
    if not ordered:
        return trace

    done_at = None
    for members, nominal in _partition(ordered, cfg):
        start = max(nominal, max(r.arrival_time + params.preprocess_ms for r in members))
        if done_at is not None:
            start = max(start, done_at)
        model_dur = iteration_time(len(members),
                                   sum(m.batch_size * params.request_bytes for m in members),
                                   params, tp)
        n_iters = max(m.actual_output_length for m in members)
        for m in members:
            ev.append(TraceEvent(start, EventKind.FUSED, m.request_id, None))
        bs = None
        if executor is not None:
            bs = _BatchStream(clock)
            for m in members:
                executor.on_fuse(m.request_id, bs.layout.fuse_request(m.request_id, 1), m)
        t = start
        for k in range(1, n_iters + 1):
            dur = model_dur
            if bs is not None:
                executor.run_iteration(bs)
                bs.iteration_index += 1
                if clock == "device":
                    dur = executor.iteration_ms()
            t = start + k * dur if clock == "cost" else t + dur
            for m in members:
                if k <= m.actual_output_length:
                    if record_tokens:
                        ev.append(TraceEvent(t, EventKind.TOKEN_GENERATED, m.request_id, k))
                    if k == m.actual_output_length:
                        ev.append(TraceEvent(t, EventKind.EVICTED, m.request_id, None))
                        if bs is not None:       # rides along as an ORPHAN row
                            slot = bs.layout.per_request_offset[m.request_id]
                            bs.layout.evict_request(m.request_id)
                            executor.on_evict(m.request_id, slot)
            ev.append(TraceEvent(t, EventKind.ITERATION_COMPLETED, None, dur))
        done_at = start + n_iters * model_dur if clock == "cost" else t
    if executor is not None:
        executor.on_drain(None)
    trace.sort()
    return trace


# --------------------------------------------------------------------------
# Concurrent instances -- one model instance per request.
#
# Drop-in for the reference's ``run_concurrent_instances`` (baselines.py:
# 130-229, contention model cost.py:112-116): an instance starts when its
# request clears preprocessing and needs ``actual_output_length`` tokens at
# its solo iteration time d; while k instances are live every one of them
# advances at 1 / (d * (1 + gamma (k - 1))) tokens per ms, re-evaluated at
# every start and finish with the fractional progress carried over.  The
# trace (cost clock) is byte-identical to the reference's
# (tests/test_baselines_golden.py).
#
# With a ``CudaExecutor`` every token of every instance is really computed:
# each instance is its own single-row stream over its own KV slot, and the
# token events are replayed in trace order as batch-1 decode steps -- so the
# instance tokens can be checked against the fused run's (greedy decoding
# does not depend on how requests are batched).

def run_concurrent_instances(requests, params: CostParams, tp: TPConfig | None = None,
                             record_tokens: bool = True, *, executor=None, clock: str = "cost",
                             max_instances: int = 64) -> Trace:
    if clock not in ("cost", "device"):
        raise InvalidParam(f"clock must be 'cost' or 'device', got {clock!r}")
    if clock == "device" and executor is None:
        raise InvalidParam("clock='device' needs an executor")
    tp = tp or TPConfig()
    from .engine import check_tp
    check_tp(tp, executor, clock)
    if clock == "device":
        return _instances_on_device(requests, params, record_tokens, executor, max_instances)
    ordered = sorted(requests, key=lambda r: (r.arrival_time, r.request_id))
    ev = []
    for r in ordered:
        ev.append(TraceEvent(r.arrival_time, EventKind.ARRIVED, r.request_id, None))
        ev.append(TraceEvent(r.arrival_time, EventKind.PREPROCESS_START, r.request_id, None))
        ev.append(TraceEvent(r.arrival_time + params.preprocess_ms, EventKind.PREPROCESS_DONE,
                             r.request_id, None))
    trace = Trace("concurrent", ev)
    if not ordered:
        return trace
    # per instance: [rid, ready, solo step time d, length, progress, time of its last token]
    inst = [[r.request_id, r.arrival_time + params.preprocess_ms,
             iteration_time(1, r.batch_size * params.request_bytes, params, tp),
             r.actual_output_length, 0.0, 0.0] for r in ordered]
    inst.sort(key=lambda x: (x[1], x[0]))
    RID, READY, D, LEN, PROG, LAST = range(6)
    live, nxt, now = [], 0, inst[0][READY]
    token_log = []                       # (time, rid, j) for the device replay

    def start_ready():
        nonlocal nxt
        while nxt < len(inst) and inst[nxt][READY] <= now:
            x = inst[nxt]
            nxt += 1
            x[LAST] = now
            live.append(x)
            ev.append(TraceEvent(now, EventKind.FUSED, x[RID], None))

    start_ready()
    while live or nxt < len(inst):
        if not live:
            now = max(now, inst[nxt][READY])
            start_ready()
        f = 1.0 + params.contention_gamma * (len(live) - 1)
        t_start = inst[nxt][READY] if nxt < len(inst) else None
        t_fin = min(now + (x[LEN] - x[PROG]) * x[D] * f for x in live)
        ends = t_start is None or t_fin <= t_start
        t_next = t_fin if ends else t_start
        finished = []
        for x in live:
            own_end = now + (x[LEN] - x[PROG]) * x[D] * f
            fin = ends and own_end == t_fin
            prog = float(x[LEN]) if fin else x[PROG] + (t_next - now) / (x[D] * f)
            last = x[LEN] if fin else math.floor(prog)
            for j in range(math.floor(x[PROG]) + 1, last + 1):
                t_j = now + (j - x[PROG]) * x[D] * f
                if record_tokens:
                    ev.append(TraceEvent(t_j, EventKind.TOKEN_GENERATED, x[RID], j))
                    ev.append(TraceEvent(t_j, EventKind.ITERATION_COMPLETED, x[RID], t_j - x[LAST]))
                token_log.append((t_j, x[RID], j))
                x[LAST] = t_j
            x[PROG] = prog
            if fin:
                finished.append(x)
        now = t_next
        for x in finished:
            live.remove(x)
            ev.append(TraceEvent(t_fin, EventKind.EVICTED, x[RID], None))
        start_ready()
    if executor is not None:
        _replay_instances(executor, ordered, token_log)
    trace.sort()
    return trace


def _replay_instances(executor, ordered, token_log) -> None:
    """Batch-1 decode steps on the device in token order, one KV slot per
    live instance (slots recycled as instances finish)."""
    length = {r.request_id: r.actual_output_length for r in ordered}
    by_rid = {r.request_id: r for r in ordered}
    streams, free, next_slot = {}, [], 0
    for _, rid, j in sorted(token_log, key=lambda e: (e[0], e[1], e[2])):
        bs = streams.get(rid)
        if bs is None:
            slot = free.pop() if free else next_slot
            if slot == next_slot:
                if next_slot >= executor.C:
                    # a second live instance would share physical slot s % C
                    raise CapacityExceeded(f"{next_slot + 1} live instances > KV pool of {executor.C} slots")
                next_slot += 1
            bs = _BatchStream("cost")
            bs.layout.slots = [Slot(None, 0)] * slot   # this instance's own KV slot
            bs.layout.buffer_offset = slot
            executor.on_fuse(rid, bs.layout.fuse_request(rid, 1), by_rid[rid])
            streams[rid] = bs
        executor.run_iteration(bs)
        bs.iteration_index += 1
        if j == length[rid]:
            slot = bs.layout.per_request_offset[rid]
            bs.layout.evict_request(rid)
            executor.on_evict(rid, slot)
            free.append(slot)
            del streams[rid]
    executor.on_drain(None)


def _instances_on_device(requests, params: CostParams, record_tokens: bool, executor,
                         max_instances: int) -> Trace:
    """Concurrent instances under the DEVICE clock: instead of
    the reference's contention model (baselines.py:130-229, cost.py:112-116)
    the instances really run side by side -- each live request is a batch-1
    decoder on its own stream and library handle (executor.instance_pool) --
    and time is the device's: every token is stamped by its step's end event
    (one device timeline for all streams), an instance starts at the first
    moment it is ready and an instance slot is free, and an idle device jumps
    to the next ready time (engine.py:200-201).  ``executor.instance_stats``
    keeps (live instances, step ms) of every step, the measured contention."""
    import time as _time

    ordered = sorted(requests, key=lambda r: (r.arrival_time, r.request_id))
    ev = []
    for r in ordered:
        ev.append(TraceEvent(r.arrival_time, EventKind.ARRIVED, r.request_id, None))
        ev.append(TraceEvent(r.arrival_time, EventKind.PREPROCESS_START, r.request_id, None))
        ev.append(TraceEvent(r.arrival_time + params.preprocess_ms, EventKind.PREPROCESS_DONE,
                             r.request_id, None))
    trace = Trace("concurrent", ev)
    if not ordered:
        return trace
    torch = __import__("torch")
    from . import executor as exmod
    cu = exmod._cuda
    pool = executor.instance_pool(min(max_instances, len(ordered)))
    ready = sorted(((r.arrival_time + params.preprocess_ms, r.request_id, r) for r in ordered),
                   key=lambda x: (x[0], x[1]))
    nxt = 0
    free_slots = list(range(executor.C))
    live = {}                      # instance index -> [rid, slot, tokens done, last time, e0, e1, request]
    stats = []
    e_start = cu.Event(enable_timing=True)
    e_start.record(pool.streams[0])
    cu.synchronize()
    t0 = _time.perf_counter()
    offset = 0.0                   # virtual - device time (idle jumps)

    def now_ms():
        return (_time.perf_counter() - t0) * 1e3 + offset

    def start(i, rid, req, at):
        slot = free_slots.pop(0)
        executor.on_fuse(rid, slot, req)
        executor._new.clear()      # instance steps carry their own prompt rows
        ev.append(TraceEvent(at, EventKind.FUSED, rid, None))
        e0, e1 = pool.step(i, rid, slot, first=True)
        live[i] = [rid, slot, 0, at, e0, e1, req, len(live) + 1]

    while live or nxt < len(ready):
        if not live and nxt < len(ready) and ready[nxt][0] > now_ms():
            offset += ready[nxt][0] - now_ms()           # idle device: jump to the next ready time
        t = now_ms()
        while nxt < len(ready) and ready[nxt][0] <= t and pool.free:
            at, rid, req = ready[nxt]
            nxt += 1
            start(pool.free.pop(0), rid, req, max(at, t))
        for i in list(live):
            x = live[i]
            if not x[5].query():
                continue
            x[5].synchronize()
            tj = e_start.elapsed_time(x[5]) + offset
            if x[2] > 0:                  # decode steps only (the first one also runs the prompt)
                stats.append((x[7], x[4].elapsed_time(x[5])))
            x[2] += 1
            rid, req = x[0], x[6]
            tj = max(tj, x[3])
            if record_tokens:
                ev.append(TraceEvent(tj, EventKind.TOKEN_GENERATED, rid, x[2]))
                ev.append(TraceEvent(tj, EventKind.ITERATION_COMPLETED, rid, tj - x[3]))
            x[3] = tj
            if x[2] == req.actual_output_length:
                ev.append(TraceEvent(tj, EventKind.EVICTED, rid, None))
                executor.on_evict(rid, x[1])
                executor._live_ctx = 0
                free_slots.append(x[1])
                pool.free.append(i)
                del live[i]
            else:
                x[4], x[5] = pool.step(i, rid, x[1], first=False)
                x[7] = len(live)
    cu.synchronize()
    executor.instance_stats = stats
    trace.sort()
    return trace
