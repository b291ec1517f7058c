"""The temporally fused decode loop -- drop-in for reference engine.py:24-207.

Same public surface (``preprocess``, ``FusionStream`` with ``now``,
``iteration_index``, ``layout``, ``active``, ``eos_at``, ``phase``,
``events``, ``pending``, ``next_ready_time``, ``try_fuse_pending``,
``step_iteration``, ``finished_all``; ``run_fusion``) and the same schedule:
admission only at iteration boundaries (inclusive tie, FIFO by (ready, id)),
an atomic iteration gives every fused request one token, then evict -> trim
-> optional Alg.1 shuffle; idle gaps are skipped.

What is new underneath:

* an ``executor`` hook.  ``None`` is the pure schedule (bit-exact with the
  reference; pinned by tests/test_engine_golden.py).  ``CudaExecutor``
  (executor.py) runs every iteration as a real decode step on the B200
  through the C-ABI and every shuffle plan as the K10 compaction kernel.
* two clocks.  ``clock="cost"`` advances ``now`` with the reference cost
  model (parity mode: identical schedule whatever the device does).
  ``clock="device"`` advances it with the CUDA-event duration of the real
  step/shuffle (performance mode: Poisson arrivals against measured time).
* O(1) host bookkeeping per row.  The reference pays a
  ``dataclasses.replace`` per row per iteration (core.py:122, ~5.6 us).
  Stop lengths are known at admission, so here ``current_iteration`` is
  derived as ``iteration_index - base`` and finishing requests are found in
  a per-iteration bucket; token events are recorded as one snapshot per
  iteration and expanded only when ``events`` is read.
"""

from __future__ import annotations

import heapq
from collections.abc import MutableMapping

from .buffer import BufferLayout, apply_shuffle, plan_shuffle
from .core import Context, Phase, Request, RuntimeInfo, advance_phase, stop_iteration
from .cost import CostParams, TPConfig, iteration_time, shuffle_time
from .errors import EmptyStream, InvalidParam
from .trace import EventKind, Trace, TraceEvent

_TOKEN = EventKind.TOKEN_GENERATED


def preprocess(request: Request, params: CostParams, now: float) -> Context:
    """A received request becomes a fusion-ready context ``preprocess_ms``
    later; no slot, no tokens yet."""
    info = RuntimeInfo(request.request_id, None, request.batch_size * params.request_bytes,
                       "gpu", request.max_output_length, 0)
    return Context(request.request_id, now + params.preprocess_ms, info)


def check_tp(tp, executor, clock: str) -> None:
    """The modelled TP degree (TPConfig, reference cost.py:26-33) and the
    executor's real one must agree whenever the device sets the clock.
    Under the cost clock the TPConfig is only a cost-model parameter, so a
    1-GPU executor may replay a modelled TP schedule (parity mode)."""
    if executor is None or tp is None:
        return
    real = getattr(executor, "tp_size", None)
    if real is None or real == tp.tp_size:
        return
    if clock == "device" or real > 1:
        raise InvalidParam(f"TPConfig.tp_size {tp.tp_size} != executor tp_size {real}")


class _ActiveTable(MutableMapping):
    """``rid -> RuntimeInfo`` in fusion order, materialised on access.

    Internally a row is [memory_offset, tensor_size, device_type,
    max_output_length, base] with current_iteration = iteration_index - base.
    """

    __slots__ = ("_s", "_rows")

    def __init__(self, stream: "FusionStream"):
        self._s = stream
        self._rows: dict = {}

    def __getitem__(self, rid):
        r = self._rows[rid]
        return RuntimeInfo(rid, r[0], r[1], r[2], r[3], self._s.iteration_index - r[4])

    def __setitem__(self, rid, info: RuntimeInfo):
        base = self._s.iteration_index - info.current_iteration
        self._rows[rid] = [info.memory_offset, info.tensor_size, info.device_type,
                           info.max_output_length, base]
        self._s._schedule_finish(rid, base, info.max_output_length)

    def __delitem__(self, rid):
        del self._rows[rid]

    def __iter__(self):
        return iter(self._rows)

    def __len__(self):
        return len(self._rows)

    def __contains__(self, rid):
        return rid in self._rows

    def __repr__(self):
        return f"_ActiveTable({dict(self.items())!r})"


class FusionStream:
    """Mutable state of one fused serving stream."""

    def __init__(self, requests, params: CostParams, tp: TPConfig,
                 shuffle_enabled: bool = True, record_tokens: bool = True,
                 slot_capacity: int | None = None, *, executor=None, clock: str = "cost",
                 max_window: int | None = None):
        if clock not in ("cost", "device"):
            raise InvalidParam(f"clock must be 'cost' or 'device', got {clock!r}")
        if clock == "device" and executor is None:
            raise InvalidParam("clock='device' needs an executor")
        check_tp(tp, executor, clock)
        self.params = params
        self.tp = tp
        self.shuffle_enabled = shuffle_enabled
        self.record_tokens = record_tokens
        self.executor = executor
        self.clock = clock
        # admission control (extension; None = reference semantics): contexts
        # stay queued while the live window already spans max_window slots,
        # i.e. while the device KV pool is full
        self.max_window = max_window
        self.now = 0.0
        self.iteration_index = 0
        self.layout = BufferLayout(capacity=slot_capacity)
        self.active = _ActiveTable(self)
        self.eos_at: dict = {}
        self.phase: dict = {}
        self.requests: dict = {}
        self._ev: list = []
        self._tok: list = []          # (position in _ev, time, rid snapshot, k)
        self._base: dict = {}         # rid -> base, kept after eviction
        self._finish_at: dict = {}    # iteration index -> [rid] in fusion order
        self._finish_of: dict = {}    # rid -> iteration index
        self.device_ms: list = []     # per-iteration device time (executor runs)
        self.widest_window = 0        # widest live window seen (rows per iteration)

        # overlapped preprocessing on the device: an executor
        # with a side-stream prefill lane starts every arrived prompt at the
        # next iteration boundary.  Under the cost clock readiness still
        # follows the model (arrival + preprocess_ms, identical schedule);
        # under the device clock a context is ready at its launch boundary
        # plus the MEASURED prefill time (``_measured_pp``).
        self._side = executor is not None and getattr(executor, "side_prefill", False)
        self._eos = getattr(executor, "eos_token", None) if executor is not None else None
        self._measured_pp = self._side and clock == "device"
        self._by_arrival = sorted(requests, key=lambda r: (r.arrival_time, r.request_id))
        self._next_launch = 0
        self._ready: list = []        # measured mode: heap of (ready, rid, ctx)
        self._admitted = 0
        pending = []
        for req in self._by_arrival:
            rid = req.request_id
            self.requests[rid] = req
            self.phase[rid] = Phase.RECEIVED
            self._emit(req.arrival_time, EventKind.ARRIVED, rid)
            self.phase[rid] = advance_phase(Phase.RECEIVED, Phase.PREPROCESSING)
            self._emit(req.arrival_time, EventKind.PREPROCESS_START, rid)
            # EOS mode (executor.eos_token): the stop is discovered on the
            # device; until then only max_output_length bounds the request
            self.eos_at[rid] = (req.max_output_length if self._eos is not None
                                else req.actual_output_length)
            if self._measured_pp:
                continue
            ctx = preprocess(req, params, req.arrival_time)
            self._emit(ctx.ready_time, EventKind.PREPROCESS_DONE, rid)
            pending.append(ctx)
        pending.sort(key=lambda c: (c.ready_time, c.request_id))
        self.pending: list = pending
        self._next_pending = 0

    # -- events ------------------------------------------------------------
    def _emit(self, time, kind, rid=None, value=None):
        self._ev.append(TraceEvent(time, kind, rid, value))

    @property
    def events(self) -> list:
        """Flat event list; per-iteration token snapshots expanded in place."""
        if self._tok:
            out = []
            prev = 0
            base = self._base
            for pos, t, rids, k in self._tok:
                out.extend(self._ev[prev:pos])
                out.extend([TraceEvent(t, _TOKEN, rid, k - base[rid]) for rid in rids])
                prev = pos
            out.extend(self._ev[prev:])
            self._ev = out
            self._tok = []
        return self._ev

    # -- queue ---------------------------------------------------------------
    def next_ready_time(self):
        if self._measured_pp:
            if not self._ready:
                self._resolve(block=True)
            return self._ready[0][0] if self._ready else None
        if self._next_pending >= len(self.pending):
            return None
        return self.pending[self._next_pending].ready_time

    def idle_advance(self) -> None:
        """Nothing fused: jump the clock to the next admissible context
        (engine.py:200-201).  With measured prefill, an idle stream first
        jumps to the next arrival and starts its prompt there."""
        while True:
            t = self.next_ready_time()
            if t is not None:
                self.now = max(self.now, t)
                return
            if self._next_launch >= len(self._by_arrival):
                raise EmptyStream("no pending contexts")
            self.now = max(self.now, self._by_arrival[self._next_launch].arrival_time)
            self._launch_prefills()

    def _launch_prefills(self) -> None:
        """Start every prompt that arrived by ``now`` on the side stream."""
        lo = self._next_launch
        hi = lo
        arr = self._by_arrival
        while hi < len(arr) and arr[hi].arrival_time <= self.now:
            hi += 1
        if hi > lo:
            self._next_launch += self.executor.launch_prefill(arr[lo:hi], self.now)

    def _resolve(self, block: bool) -> None:
        for rid, ready in self.executor.poll_prefill(block):
            self._emit(ready, EventKind.PREPROCESS_DONE, rid)
            req = self.requests[rid]
            info = RuntimeInfo(rid, None, req.batch_size * self.params.request_bytes, "gpu",
                               req.max_output_length, 0)
            heapq.heappush(self._ready, (ready, rid, Context(rid, ready, info)))

    def _schedule_finish(self, rid, base, max_out):
        old = self._finish_of.pop(rid, None)
        if old is not None:
            self._finish_at[old].remove(rid)
        at = base + stop_iteration(self.eos_at[rid], max_out) - 1
        self._finish_of[rid] = at
        self._finish_at.setdefault(at, []).append(rid)
        self._base[rid] = base

    def _next_admissible(self):
        """The next context in (ready, id) order if it is ready by ``now``."""
        if self._measured_pp:
            if self._ready and self._ready[0][0] <= self.now:
                return heapq.heappop(self._ready)[2]
            return None
        pend = self.pending
        if self._next_pending < len(pend) and pend[self._next_pending].ready_time <= self.now:
            self._next_pending += 1
            return pend[self._next_pending - 1]
        return None

    def try_fuse_pending(self) -> int:
        """Admit, in FIFO order, every context ready at or before ``now``."""
        n = 0
        cap = self.max_window
        if self._side:
            self._launch_prefills()
            if self._measured_pp:
                self._resolve(block=False)
        while True:
            if cap is not None and self.layout.buffer_size >= cap:
                break
            ctx = self._next_admissible()
            if ctx is None:
                break
            self._admitted += 1
            rid = ctx.request_id
            slot = self.layout.fuse_request(rid, ctx.runtime.tensor_size)
            rt = ctx.runtime
            self.active[rid] = RuntimeInfo(rid, slot, rt.tensor_size, rt.device_type,
                                           rt.max_output_length, rt.current_iteration)
            ph = advance_phase(self.phase[rid], Phase.READY_FOR_FUSION)
            self.phase[rid] = advance_phase(ph, Phase.RUNNING)
            self._emit(self.now, EventKind.FUSED, rid)
            if self.executor is not None:
                self.executor.on_fuse(rid, slot, self.requests.get(rid))
            n += 1
        return n

    # -- the atomic iteration --------------------------------------------------
    def step_iteration(self) -> None:
        """One atomic iteration (engine.py:128-177).  With an executor the
        step is launched first; the end-of-iteration layout work (evictions,
        trims, the shuffle plan and its K10 launch) needs no clock and runs on
        the host while the step executes; the clock advance and the events
        follow once the step's (measured or modelled) duration is known."""
        if not self.active:
            raise EmptyStream("no fused requests to iterate")
        lay = self.layout
        if lay.buffer_size > self.widest_window:
            self.widest_window = lay.buffer_size
        ex = self.executor
        dev_clock = self.clock == "device"
        if ex is not None:
            ex.run_iteration(self)            # launched (device clock: timed, read below)
        if not dev_clock:
            duration = iteration_time(len(self.active), lay.live_bytes(), self.params, self.tp)
        snap = tuple(self.active._rows) if self.record_tokens else None
        it = self.iteration_index

        if self._eos is not None:
            # data-dependent stop: a request whose token of this iteration is
            # EOS finishes now -- record_token's eos_at (core.py:108-123)
            # becomes the iteration count at which the token appeared
            for rid in ex.eos_hits():
                base = self._base[rid]
                if self._finish_of.get(rid) != it:
                    self.eos_at[rid] = it - base + 1
                    self._schedule_finish(rid, base, self.requests[rid].max_output_length)
        done = self._finish_at.pop(it, ())
        rows = self.active._rows
        for rid in done:
            slot = lay.per_request_offset[rid]
            lay.evict_request(rid)
            del rows[rid]
            del self._finish_of[rid]
            self.phase[rid] = advance_phase(self.phase[rid], Phase.FINISHED)
            if ex is not None:
                ex.on_evict(rid, slot)
        self.iteration_index += 1

        plan = None
        if self.shuffle_enabled:
            lay.trim_boundaries()
            if done and lay.has_interior_holes():
                on_device = ex is not None and getattr(ex, "device_plan", False)
                if on_device:
                    # planned and executed on the device (csrc/planner.cu + K10);
                    # the host only mirrors the returned plan
                    plan = ex.shuffle_on_device(lay)
                else:
                    plan = plan_shuffle(lay)
                if plan.moves:
                    apply_shuffle(lay, plan)
                    if not on_device and ex is not None:
                        ex.on_shuffle(plan, timed=dev_clock)
                else:
                    plan = None
        else:
            lay.trim_leading()

        if dev_clock:
            duration = ex.iteration_ms()
            self.device_ms.append(duration)
        self.now += duration
        now = self.now
        if snap is not None:
            self._tok.append((len(self._ev), now, snap, it + 1))
        for rid in done:
            self._emit(now, EventKind.EVICTED, rid)
        self._emit(now, EventKind.ITERATION_COMPLETED, None, duration)
        if plan is not None:
            self.now += ex.shuffle_ms() if dev_clock else shuffle_time(plan.total_bytes_moved, self.params)
            self._emit(self.now, EventKind.SHUFFLE_EXECUTED, None, plan.total_bytes_moved)

    def finished_all(self) -> bool:
        if self._measured_pp:
            return not self.active and self._admitted >= len(self.requests)
        return not self.active and self._next_pending >= len(self.pending)


def run_fusion(requests, params: CostParams, tp: TPConfig | None = None,
               shuffle_enabled: bool = True, record_tokens: bool = True, *,
               executor=None, clock: str = "cost", max_window: int | None = None) -> Trace:
    """Serve every request to completion on one fused stream."""
    stream = FusionStream(requests, params, tp or TPConfig(), shuffle_enabled=shuffle_enabled,
                          record_tokens=record_tokens, executor=executor, clock=clock,
                          max_window=max_window)
    drive(stream)
    trace = Trace("fusion" if shuffle_enabled else "fusion_noshuffle", stream.events)
    trace.sort()
    return trace


def drive(stream: FusionStream) -> FusionStream:
    """The loop of engine.py:199-203, idle jump included."""
    while not stream.finished_all():
        if not stream.active:
            stream.idle_advance()
        stream.try_fuse_pending()
        stream.step_iteration()
    if stream.executor is not None:
        stream.executor.on_drain(stream)
    return stream
