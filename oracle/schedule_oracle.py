"""CPU oracle for the fused-stream SCHEDULE (test infrastructure only).

THIS IS A CHECKER, NOT PRODUCT CODE.  Only ``tests/``,
``__graft_entry__.smoke()`` and ``bench.py``'s ``cpu_baseline`` /
``--impl reference`` legs may import it.  The product path
(``paper_2305_13484_b200``) never imports anything under ``oracle/``.

It restates, in a deliberately plain procedural form, the integer/index
algorithm of the reference simulator ``fusionsim`` (mounted read-only at
/root/reference/pkg/src/fusionsim) for the temporally fused decode loop:

  * seeded generator ............ rng.py:25-67   (splitmix64 + xorshift64*)
  * arrival / length sampling ... arrivals.py:60-93, scenario.py:97-124
  * preprocess .................. engine.py:24-42
  * admission ................... engine.py:97-124, buffer.py:170-186
  * one atomic iteration ........ engine.py:128-177, core.py:108-123
  * slot eviction / trims ....... buffer.py:188-223
  * Algorithm 1 window search ... buffer.py:59-88
  * shuffle plan / apply ........ buffer.py:226-278
  * virtual clock ............... cost.py:73-123
  * loop driver + idle jump ..... engine.py:183-207
  * trace formatting ............ trace.py:41-54

Parity status: PINNED.  tests/golden/ holds vectors produced by running the
reference itself (tests/golden/gen_golden.py imports /root/reference in the
build container); tests/test_oracle_golden.py checks this module against
every one of them.

Output of :func:`fused_schedule` is a ``Schedule``: the flat event list
(same tuples as the reference ``TraceEvent``) plus one ``IterRecord`` per
iteration describing exactly what the device must execute: the window rows
(slot -> request or hole), admissions, the finished set and the shuffle
moves.  The model-level oracle (model_oracle.py) replays these records.
"""

from __future__ import annotations

import math
from dataclasses import dataclass, field

U64 = (1 << 64) - 1
GOLDEN_GAMMA = 0x9E3779B97F4A7C15
XS_MULT = 0x2545F4914F6CDD1D

# event kind strings, identical to trace.py:15-23 values
ARRIVED = "arrived"
PP_START = "preprocess_start"
PP_DONE = "preprocess_done"
FUSED = "fused"
TOKEN = "token"
EVICTED = "evicted"
SHUFFLE = "shuffle"
ITERATION = "iteration"


# --------------------------------------------------------------------------
# generator (rng.py:25-67)
# --------------------------------------------------------------------------
def mix64(v: int) -> int:
    """One splitmix64 output step applied to v (rng.py:25-30)."""
    v = (v + GOLDEN_GAMMA) & U64
    v = ((v ^ (v >> 30)) * 0xBF58476D1CE4E5B9) & U64
    v = ((v ^ (v >> 27)) * 0x94D049BB133111EB) & U64
    return v ^ (v >> 31)


def seed_for(seed: int, stream: int) -> int:
    """rng.py:33-35."""
    return mix64((seed & U64) ^ mix64(stream & U64))


class XorStar:
    """xorshift64* (rng.py:38-67); state seeded through seed_for(seed, stream)."""

    def __init__(self, seed: int, stream: int = 0):
        s = seed_for(seed, stream)
        self.s = s if s else GOLDEN_GAMMA

    def u64(self) -> int:
        s = self.s
        s ^= s >> 12
        s ^= (s << 25) & U64
        s ^= s >> 27
        self.s = s
        return (s * XS_MULT) & U64

    def unit(self) -> float:
        return (self.u64() >> 11) * (1.0 / 9007199254740992.0)

    def expo(self, mean: float) -> float:
        return -mean * math.log1p(-self.unit())

    def int_in(self, lo: int, hi: int) -> int:
        return lo + int(self.unit() * (hi - lo + 1))


# --------------------------------------------------------------------------
# workload (arrivals.py:60-93, scenario.py:97-124)
# --------------------------------------------------------------------------
@dataclass(frozen=True)
class Req:
    rid: int
    batch: int
    input_len: int
    max_out: int
    actual_out: int
    arrival: float


def arrivals_poisson(n: int, mean_ms: float, seed: int, start: float = 0.0) -> list[float]:
    g = XorStar(seed)
    out = [start]
    t = start
    for _ in range(1, n):
        t += g.expo(mean_ms)
        out.append(t)
    return out


def arrivals_constant(n: int, gap_ms: float, start: float = 0.0) -> list[float]:
    return [start + i * gap_ms for i in range(n)]


def lengths_uniform(n: int, lo: int, hi: int, seed: int) -> list[int]:
    g = XorStar(seed)
    return [g.int_in(lo, hi) for _ in range(n)]


def scenario_requests(n, *, poisson_mean_ms=None, constant_gap_ms=None,
                      lengths=(1, 1), max_out=1, input_len=32, batch=1,
                      seed=0) -> list[Req]:
    """scenario.build_requests: arrivals use seed_for(seed, 1) which the
    generator derives AGAIN with stream 0 (scenario.py:103 + rng.py:42);
    lengths use seed_for(seed, 2) (scenario.py:112)."""
    if poisson_mean_ms is not None:
        times = arrivals_poisson(n, poisson_mean_ms, seed_for(seed, 1))
    else:
        times = arrivals_constant(n, constant_gap_ms)
    lo, hi = lengths
    if lo == hi:
        lens = [lo] * n
    else:
        lens = lengths_uniform(n, lo, hi, seed_for(seed, 2))
    return [Req(i, batch, input_len, max_out, lens[i], times[i]) for i in range(n)]


def prompt_tokens(n: int, input_len: int, vocab: int, seed: int) -> list[list[int]]:
    """Synthetic prompts (stream tag 3, unused by the reference)."""
    g = XorStar(seed_for(seed, 3))
    return [[g.int_in(0, vocab - 1) for _ in range(input_len)] for _ in range(n)]


# --------------------------------------------------------------------------
# cost model (cost.py:36-123)
# --------------------------------------------------------------------------
@dataclass(frozen=True)
class Cost:
    base_iteration_ms: float = 6000.0 / 512.0
    marginal_per_request_ms: float = 0.05
    capacity: int = 4
    preprocess_ms: float = 6000.0 / 512.0
    alpha_intra_ms: float = 0.02
    alpha_inter_ms: float = 0.2
    beta_intra_ms_per_byte: float = 2.0e-5
    beta_inter_ms_per_byte: float = 8.0e-5
    memcpy_beta_ms_per_byte: float = 1.0e-6
    contention_gamma: float = 0.35
    request_bytes: int = 1_000_000


def step_ms(n_active: int, live: int, c: Cost, tp: int, inter: bool) -> float:
    """cost.py:89-109 with comm_time cost.py:73-86 inlined in the same
    floating-point operation order (2*call + call)."""
    t = c.base_iteration_ms + c.marginal_per_request_ms * max(0, n_active - c.capacity)
    if tp > 1:
        a, b = ((c.alpha_inter_ms, c.beta_inter_ms_per_byte) if inter
                else (c.alpha_intra_ms, c.beta_intra_ms_per_byte))
        call = a + b * (live / tp)
        t += 2.0 * call + call
    return t


# --------------------------------------------------------------------------
# Algorithm 1 (buffer.py:59-88) and the brute-force cross-check (:99-122)
# --------------------------------------------------------------------------
def alg1(arr) -> int:
    k = sum(1 for v in arr if v)
    total = sum(v for v in arr if v)
    inside = sum(arr[:k])
    best = total - inside
    off = 0
    for i in range(k, len(arr)):
        inside += arr[i] - arr[i - k]
        if total - inside < best:          # strict: earliest tie wins (:85)
            best = total - inside
            off = i - k + 1
    return off


def alg1_brute(arr) -> tuple[int, int]:
    k = sum(1 for v in arr if v)
    if k == 0:
        return 0, 0
    total = sum(arr)
    best = None
    off = 0
    for o in range(len(arr) - k + 1):
        cst = total - sum(arr[o:o + k])
        if best is None or cst < best:
            best, off = cst, o
    return off, best


# --------------------------------------------------------------------------
# the fused loop
# --------------------------------------------------------------------------
@dataclass
class IterRecord:
    index: int
    t_start: float                 # clock when the iteration starts
    duration: float                # clock advance for the iteration
    admitted: list                 # [(rid, logical_slot)] fused at this boundary
    window_offset: int             # live window BEFORE the iteration
    rows: list                     # [(logical_slot, rid or None)] window rows
    finished: list                 # rids that produced their last token
    moves: list                    # [(rid, src_slot, dst_slot, size)]
    shuffle_bytes: int
    t_end: float                   # clock after boundary work
    window_after: tuple            # (offset, size) after boundary work


@dataclass
class Schedule:
    events: list = field(default_factory=list)    # (time, kind, rid, value)
    iters: list = field(default_factory=list)

    def trace_lines(self) -> list[str]:
        """trace.py:47-54 formatting."""
        out = []
        for t, k, r, v in self.events:
            out.append(f"{t:.6f}\t{k}\t{'-' if r is None else r}\t{'-' if v is None else repr(v)}")
        return out


def fused_schedule(reqs: list[Req], cost: Cost = Cost(), tp: int = 1,
                   inter: bool = False, shuffle: bool = True,
                   record_tokens: bool = True) -> Schedule:
    sch = Schedule()
    ev = sch.events
    # engine.py:72-84 -- lifecycle prefix and the FIFO of contexts
    ctxs = []
    stop = {}
    for r in sorted(reqs, key=lambda q: (q.arrival, q.rid)):
        ev.append((r.arrival, ARRIVED, r.rid, None))
        ev.append((r.arrival, PP_START, r.rid, None))
        ready = r.arrival + cost.preprocess_ms
        ev.append((ready, PP_DONE, r.rid, None))
        ctxs.append((ready, r.rid, r.batch * cost.request_bytes))
        stop[r.rid] = min(r.actual_out, r.max_out)        # core.py:117
    ctxs.sort(key=lambda c: (c[0], c[1]))

    occ: list = []          # slot -> rid or None
    sz: list = []           # slot -> byte size (kept after eviction)
    off = 0
    n = 0                   # window length
    where: dict = {}        # rid -> slot
    active: dict = {}       # rid -> tokens so far (insertion order = event order)
    now = 0.0
    nxt = 0
    it = 0

    while active or nxt < len(ctxs):
        if not active:                                       # idle jump
            now = max(now, ctxs[nxt][0])
        admitted = []
        while nxt < len(ctxs) and ctxs[nxt][0] <= now:       # inclusive boundary
            _, rid, size = ctxs[nxt]
            nxt += 1
            idx = off + n
            if idx < len(occ):
                occ[idx] = rid
                sz[idx] = size
            else:
                occ.append(rid)
                sz.append(size)
            n += 1
            where[rid] = idx
            active[rid] = 0
            ev.append((now, FUSED, rid, None))
            admitted.append((rid, idx))

        rows = [(s, occ[s]) for s in range(off, off + n)]
        live = sum(sz[off:off + n])
        dur = step_ms(len(active), live, cost, tp, inter)
        t0 = now
        now += dur
        done = []
        for rid in active:
            active[rid] += 1
            if record_tokens:
                ev.append((now, TOKEN, rid, active[rid]))
            if active[rid] == stop[rid]:
                done.append(rid)
        for rid in done:
            occ[where.pop(rid)] = None
            del active[rid]
            ev.append((now, EVICTED, rid, None))
        ev.append((now, ITERATION, None, dur))

        moves = []
        moved = 0
        win0 = off
        if shuffle:
            while n and occ[off] is None:
                off += 1
                n -= 1
            while n and occ[off + n - 1] is None:
                n -= 1
            if done and n > len(where):
                arr = [sz[s] if occ[s] is not None else 0 for s in range(off, off + n)]
                lo = off + alg1(arr)
                hi = lo + len(where)
                src = [s for s in range(off, off + n) if occ[s] is not None and not lo <= s < hi]
                dst = [s for s in range(off, off + n) if occ[s] is None and lo <= s < hi]
                for a, b in zip(src, dst):
                    moves.append((occ[a], a, b, sz[a]))
                if moves:
                    for rid, a, b, size in moves:
                        occ[b] = rid
                        sz[b] = size
                        occ[a] = None
                        where[rid] = b
                    off, n = lo, len(where)
                    moved = sum(m[3] for m in moves)
                    now += cost.memcpy_beta_ms_per_byte * moved
                    ev.append((now, SHUFFLE, None, moved))
        else:
            while n and occ[off] is None:
                off += 1
                n -= 1

        sch.iters.append(IterRecord(it, t0, dur, admitted, win0, rows, done,
                                    moves, moved, now, (off, n)))
        it += 1

    ev.sort(key=lambda e: e[0])          # stable, trace.py:41-42
    return sch
