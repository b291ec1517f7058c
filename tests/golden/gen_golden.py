"""Generate golden vectors by running the REFERENCE simulator itself.

Runs only in the build container, where the reference is mounted read-only
at /root/reference (it does not exist on the GPU box, so nothing at test
time imports it).  Re-run with

    PYTHONDONTWRITEBYTECODE=1 python tests/golden/gen_golden.py

The outputs are small JSON(.gz) fixtures next to this script:

  rng.json            splitmix/xorshift64* streams, floats, ints, exponentials
                      (reference rng.py:25-67)
  alg1.json           Algorithm 1 offsets on hand, exhaustive-binary and
                      random weighted arrays (buffer.py:59-88, oracle.py:47-64)
  plans.json          plan_shuffle move lists on randomized layouts
                      (buffer.py:226-278)
  requests.json       build_requests outputs for the bench scenarios
                      (scenario.py:97-124)
  schedules.json.gz   per-iteration fused-loop dumps + full-trace digests for
                      hand cases, C1-C4 and randomized prop_helpers-style
                      cases (engine.py:128-207)
  dynbatch.json.gz    run_dynamic_batching traces (baselines.py:51-127)
  concurrent.json.gz  run_concurrent_instances traces (baselines.py:130-229)
  suite.csv           the results CSV of a scenario grid (suite.py:23-54,
                      137-172): every discipline, constant / Poisson
                      arrivals, fixed / uniform lengths, TP 1 / 2, 1-3 seeds
"""

from __future__ import annotations

import gzip
import hashlib
import json
import os
import sys

REF = "/root/reference/pkg/src"
HERE = os.path.dirname(os.path.abspath(__file__))
sys.dont_write_bytecode = True
sys.path.insert(0, REF)

from fusionsim import buffer as rbuf  # noqa: E402
from fusionsim import oracle as rorc  # noqa: E402
from fusionsim.core import Request  # noqa: E402
from fusionsim.cost import CostParams, TPConfig, Placement  # noqa: E402
from fusionsim.engine import FusionStream, run_fusion  # noqa: E402
from fusionsim.rng import Xorshift64Star, derive_seed  # noqa: E402
from fusionsim.scenario import (  # noqa: E402
    Discipline, PoissonArrival, ConstantArrival, Scenario, build_requests,
)
from fusionsim.arrivals import UniformLength, FixedLength  # noqa: E402
from fusionsim.trace import EventKind, Trace  # noqa: E402


def _dump(name, obj, gz=False):
    path = os.path.join(HERE, name)
    data = json.dumps(obj, sort_keys=True, separators=(",", ":")).encode()
    if gz:
        with gzip.GzipFile(path, "wb", mtime=0) as f:
            f.write(data)
    else:
        with open(path, "wb") as f:
            f.write(data)
    print(f"wrote {name}: {len(data)} bytes")


# ---------------------------------------------------------------- rng
def gen_rng():
    seeds = [0, 1, 2, 3, 7, 42, 1234, 2**63 + 5, 2**64 - 1]
    out = {"derive": [], "streams": []}
    for s in seeds:
        for st in range(5):
            out["derive"].append([s, st, derive_seed(s, st)])
    for s in seeds:
        for st in (0, 1, 3):
            g = Xorshift64Star(s, st)
            u = [g.next_u64() for _ in range(16)]
            f = [g.next_float().hex() for _ in range(8)]
            i = [g.uniform_int(0, 50256) for _ in range(8)] + [g.uniform_int(128, 1024) for _ in range(8)]
            e = [g.exponential(20.0).hex() for _ in range(8)]
            out["streams"].append({"seed": s, "stream": st, "u64": u, "float": f, "int": i, "exp": e})
    _dump("rng.json", out)


# ---------------------------------------------------------------- alg1
def gen_alg1():
    cases = []
    hand = [[], [0, 0, 0], [3], [0, 1, 1], [1, 0, 1], [2, 0, 0, 2], [5, 0, 2],
            [1, 0, 1, 1, 0, 1], [0, 0, 4, 4, 0], [1, 0, 2, 0, 1], [3, 0, 3, 0, 3]]
    arrays = hand + [list(a) for L in range(0, 11) for a in rorc.all_binary_arrays(L)]
    arrays += [list(a) for a in rorc.random_weighted_arrays(1000, seed=7)]
    # long weighted windows like the C3 shuffle (window ~512)
    g = Xorshift64Star(99)
    for _ in range(50):
        n = g.uniform_int(100, 600)
        arrays.append([0 if g.next_float() < 0.1 else g.uniform_int(1, 10**6) for _ in range(n)])
    for a in arrays:
        off = rbuf.find_shuffled_memory_region(a)
        cases.append([a, off, rbuf.window_move_cost(a, off)])
    _dump("alg1.json", {"cases": cases})


# ---------------------------------------------------------------- plans
def gen_plans():
    g = Xorshift64Star(2024)
    out = []
    for _ in range(300):
        lay = rbuf.BufferLayout()
        n = g.uniform_int(1, 40)
        ops = []
        for rid in range(n):
            lay.fuse_request(rid, g.uniform_int(1, 1000))
        for rid in range(n):
            if g.next_float() < 0.4:
                lay.evict_request(rid)
                ops.append(rid)
        lay.trim_boundaries()
        sizes = [lay.slots[i].size for i in range(len(lay.slots))]
        plan = rbuf.plan_shuffle(lay)
        out.append({
            "sizes": sizes, "evicted": ops,
            "window": [lay.buffer_offset, lay.buffer_size],
            "moves": [[m.request_id, m.src_slot, m.dst_slot, m.size] for m in plan.moves],
            "plan_window": [plan.window_offset, plan.window_len],
            "bytes": plan.total_bytes_moved,
        })
    _dump("plans.json", {"cases": out})


# ---------------------------------------------------------------- scenarios
SCEN = {
    # name: (n, mean_ms, lo, hi, max_out, input_len)
    "c1": (32, 20.0, 8, 64, 64, 16),
    "c2": (128, 20.0, 32, 512, 512, 32),
    "c3": (512, 20.0, 128, 1024, 1024, 32),
    "c4": (64, 20.0, 128, 1024, 1024, 32),
}


def scen(name, seed, disc=Discipline.FUSION, tp=1):
    n, mean, lo, hi, mx, il = SCEN[name]
    sc = Scenario(scenario_id=name, discipline=disc, n_requests=n,
                  arrival=PoissonArrival(mean), lengths=UniformLength(lo, hi),
                  max_output_length=mx, input_len=il, tp=TPConfig(tp_size=tp))
    return build_requests(sc, seed)


def gen_requests():
    out = {}
    for name in SCEN:
        for seed in (1, 2, 5):
            reqs = scen(name, seed)
            out[f"{name}/{seed}"] = [[r.request_id, r.batch_size, r.input_len, r.max_output_length,
                                      r.actual_output_length, r.arrival_time.hex()] for r in reqs]
    # constant-arrival scenario
    sc = Scenario(scenario_id="k", discipline=Discipline.FUSION, n_requests=16,
                  arrival=ConstantArrival(20.0), lengths=UniformLength(128, 1792),
                  max_output_length=1792)
    out["const/3"] = [[r.request_id, r.batch_size, r.input_len, r.max_output_length,
                       r.actual_output_length, r.arrival_time.hex()] for r in build_requests(sc, 3)]
    _dump("requests.json", out)


def stepwise_dump(requests, params, tp, shuffle, record_tokens=True):
    """Drive the reference FusionStream by hand (engine.py:199-203) and
    record, per iteration, what the device must execute."""
    st = FusionStream(requests, params, tp, shuffle_enabled=shuffle, record_tokens=record_tokens)
    lines = []
    it = 0
    while not st.finished_all():
        if not st.active:
            st.now = max(st.now, st.next_ready_time())
        before = set(st.active)
        st.try_fuse_pending()
        admitted = [[rid, st.layout.per_request_offset[rid]] for rid in st.active if rid not in before]
        lay = st.layout
        win0 = lay.buffer_offset
        rows = [(-1 if lay.slots[s].occupant is None else lay.slots[s].occupant)
                for s in range(lay.buffer_offset, lay.buffer_offset + lay.buffer_size)]
        offs = dict(lay.per_request_offset)
        t0 = st.now
        ne = len(st.events)
        st.step_iteration()
        new = st.events[ne:]
        fin = [e.request_id for e in new if e.kind is EventKind.EVICTED]
        dur = [e.value for e in new if e.kind is EventKind.ITERATION_COMPLETED][0]
        sh = [e.value for e in new if e.kind is EventKind.SHUFFLE_EXECUTED]
        moves = sorted([[rid, offs[rid], s, lay.slots[s].size]
                        for rid, s in lay.per_request_offset.items() if offs[rid] != s],
                       key=lambda m: m[1])
        lines.append(iter_line(it, t0, dur, win0, rows, admitted, fin, moves,
                               sh[0] if sh else 0, st.now, (lay.buffer_offset, lay.buffer_size)))
        it += 1
    tr = Trace("x", st.events)
    tr.sort()
    return lines, tr.format_lines()


def iter_line(it, t0, dur, win0, rows, admitted, fin, moves, moved, t1, after):
    """Canonical per-iteration text (shared with tests/schedule_dump.py)."""
    return "|".join([str(it), float(t0).hex(), float(dur).hex(), str(win0),
                     ",".join(map(str, rows)),
                     ";".join(f"{a}@{b}" for a, b in admitted),
                     ",".join(map(str, fin)),
                     ";".join(f"{r}:{a}>{b}:{s}" for r, a, b, s in moves),
                     str(moved), float(t1).hex(), f"{after[0]}+{after[1]}"])


def sha(lines):
    h = hashlib.sha256()
    for ln in lines:
        h.update(ln.encode())
        h.update(b"\n")
    return h.hexdigest()


TIGHT = dict(base_iteration_ms=10.0, marginal_per_request_ms=0.0, preprocess_ms=10.0,
             alpha_intra_ms=0.0, beta_intra_ms_per_byte=2.0**-10,
             memcpy_beta_ms_per_byte=2.0**-10, request_bytes=100)


def _req(rid, arrival, length, max_out=None, batch=1, input_len=32):
    return Request(rid, batch, input_len, max_out or max(length, 1), length, arrival)


def random_cost(g):
    beta = 1.0e-5 + 4.0e-5 * g.next_float()
    return dict(base_iteration_ms=5.0 + 10.0 * g.next_float(),
                marginal_per_request_ms=0.2 * g.next_float(),
                capacity=g.uniform_int(2, 6), preprocess_ms=20.0 * g.next_float(),
                alpha_intra_ms=0.05 * g.next_float(), beta_intra_ms_per_byte=beta,
                memcpy_beta_ms_per_byte=beta / 4.0 * g.next_float(),
                contention_gamma=g.next_float(), request_bytes=g.uniform_int(50_000, 2_000_000))


def random_requests(g, n=None):
    n = n or g.uniform_int(1, 12)
    t = 0.0
    out = []
    for rid in range(n):
        t += g.next_float() * 60.0
        out.append(Request(rid, g.uniform_int(1, 2), g.uniform_int(1, 64), 40,
                           g.uniform_int(1, 30), t))
    return out


def req_json(reqs):
    return [[r.request_id, r.batch_size, r.input_len, r.max_output_length,
             r.actual_output_length, r.arrival_time.hex()] for r in reqs]


def gen_schedules():
    cases = []

    def add(name, reqs, cost, tp, shuffle, record_tokens=True, keep_lines=True, placement="intra"):
        params = CostParams(**cost)
        tpc = TPConfig(tp_size=tp, placement=Placement(placement))
        lines, trace = stepwise_dump(reqs, params, tpc, shuffle, record_tokens)
        ref = run_fusion(reqs, params, tpc, shuffle_enabled=shuffle, record_tokens=record_tokens)
        assert ref.format_lines() == trace, name
        cases.append({
            "name": name, "requests": req_json(reqs), "cost": {k: (v.hex() if isinstance(v, float) else v)
                                                                for k, v in cost.items()},
            "tp": tp, "placement": placement, "shuffle": shuffle, "record_tokens": record_tokens,
            "n_iters": len(lines), "iter_sha": sha(lines), "trace_sha": sha(trace),
            "n_events": len(trace),
            "iters": lines if keep_lines else lines[:40],
            "trace_head": trace[:60],
        })

    # hand cases from the reference engine tests (test_engine.py:43-221)
    add("single512", [_req(0, 0.0, 512, 512)], {}, 1, True)
    add("eos3", [_req(0, 0.0, 3, 512)], TIGHT, 1, True)
    add("boundary", [_req(0, 0.0, 5), _req(1, 10.0, 2), _req(2, 15.0, 1)], TIGHT, 1, True)
    add("fifo", [_req(0, 0.0, 3), _req(1, 3.0, 3), _req(2, 7.0, 3)], TIGHT, 1, True)
    add("idle", [_req(0, 0.0, 2), _req(1, 100.0, 1)], TIGHT, 1, True)
    for lens in ([3, 1, 3], [3, 3, 1], [1, 3, 3]):
        for sh in (True, False):
            add(f"orphan{lens}{sh}", [_req(i, 0.0, n) for i, n in enumerate(lens)], TIGHT, 2, sh)
    add("capacity", [_req(i, 0.0, 2) for i in range(6)],
        dict(base_iteration_ms=10.0, marginal_per_request_ms=0.5, capacity=4, preprocess_ms=10.0), 1, True)
    add("lifecycle", [_req(i, 5.0 * i, 4 + i) for i in range(4)], TIGHT, 1, True)
    add("notokens", [_req(i, 11.0 * i, 9) for i in range(4)], TIGHT, 2, True, record_tokens=False)
    add("inter", [_req(i, 3.0 * i, 5 + (i % 3)) for i in range(6)], TIGHT, 2, True, placement="inter")

    # bench scenarios (default CostParams)
    for name, tps in (("c1", (1,)), ("c2", (1, 2)), ("c3", (1, 8)), ("c4", (4,))):
        for tp in tps:
            for sh in (True, False):
                reqs = scen(name, 1)
                big = name in ("c3",) or (name == "c2" and tp == 2) or name == "c4"
                add(f"{name}/tp{tp}/{'on' if sh else 'off'}", reqs, {}, tp, sh,
                    record_tokens=True, keep_lines=not big)

    # randomized (prop_helpers.py:21-59 style)
    g = Xorshift64Star(31337)
    for i in range(120):
        cost = random_cost(g)
        reqs = random_requests(g)
        tp = 2 if g.uniform_int(0, 1) else 1
        sh = bool(i % 3)
        add(f"rand{i}", reqs, cost, tp, sh)

    _dump("schedules.json.gz", {"cases": cases}, gz=True)


def gen_dynbatch():
    """run_dynamic_batching traces (baselines.py:51-127)."""
    from fusionsim.baselines import BatchWindowConfig, run_dynamic_batching
    cases = []

    def add(name, reqs, window, max_batch, cost, tp=1, record_tokens=True):
        tr = run_dynamic_batching(reqs, BatchWindowConfig(window, max_batch), CostParams(**cost),
                                  TPConfig(tp_size=tp), record_tokens=record_tokens).format_lines()
        cases.append({"name": name, "requests": req_json(reqs), "window": window,
                      "max_batch": max_batch,
                      "cost": {k: (v.hex() if isinstance(v, float) else v) for k, v in cost.items()},
                      "tp": tp, "record_tokens": record_tokens, "trace_sha": sha(tr),
                      "n_events": len(tr), "trace_head": tr[:80]})

    # reference tests/test_baselines.py worked examples
    add("worked", [_req(0, 0.0, 3), _req(1, 100.0, 2), _req(2, 510.0, 4)], 500.0, None, {})
    add("maxbatch", [_req(i, 1.0 * i, 2 + i) for i in range(5)], 100.0, 2, TIGHT)
    add("zero_window", [_req(i, 7.0 * i, 3) for i in range(4)], 0.0, None, TIGHT)
    add("tp2", [_req(i, 13.0 * i, 4 + i % 3) for i in range(6)], 25.0, 3, TIGHT, tp=2)
    for lam in (1, 4, 16, 64):
        n, mean, lo, hi, mx, il = SCEN["c3"]
        sc = Scenario(scenario_id="c5", discipline=Discipline.DYNAMIC_BATCHING, n_requests=48,
                      arrival=PoissonArrival(1000.0 / lam), lengths=UniformLength(lo, hi),
                      max_output_length=mx, input_len=il, window_ms=50.0)
        add(f"c5/lam{lam}", build_requests(sc, 1), 50.0, None, {}, record_tokens=lam != 64)
    g = Xorshift64Star(777)
    for i in range(40):
        cost = random_cost(g)
        reqs = random_requests(g)
        add(f"rand{i}", reqs, 60.0 * g.next_float(), g.uniform_int(1, 4) if i % 2 else None, cost,
            tp=2 if i % 3 == 0 else 1)
    _dump("dynbatch.json.gz", {"cases": cases}, gz=True)


def gen_concurrent():
    """run_concurrent_instances traces (baselines.py:130-229, cost.py:112-116)."""
    from fusionsim.baselines import run_concurrent_instances
    cases = []

    def add(name, reqs, cost, tp=1, record_tokens=True):
        tr = run_concurrent_instances(reqs, CostParams(**cost), TPConfig(tp_size=tp),
                                      record_tokens=record_tokens).format_lines()
        cases.append({"name": name, "requests": req_json(reqs),
                      "cost": {k: (v.hex() if isinstance(v, float) else v) for k, v in cost.items()},
                      "tp": tp, "record_tokens": record_tokens, "trace_sha": sha(tr),
                      "n_events": len(tr), "trace_head": tr[:80]})

    add("single", [_req(0, 0.0, 3)], {})
    add("overlap", [_req(0, 0.0, 4), _req(1, 1.0, 2), _req(2, 2.5, 5)], TIGHT)
    add("same_ready", [_req(i, 0.0, 2 + i) for i in range(4)], TIGHT)
    add("idle_gap", [_req(0, 0.0, 2), _req(1, 1000.0, 3)], {})
    add("tp2", [_req(i, 5.0 * i, 3 + i % 4) for i in range(7)], TIGHT, tp=2)
    for lam in (1, 16, 64):
        n, mean, lo, hi, mx, il = SCEN["c3"]
        sc = Scenario(scenario_id="c5", discipline=Discipline.CONCURRENT, n_requests=32,
                      arrival=PoissonArrival(1000.0 / lam), lengths=UniformLength(lo, hi),
                      max_output_length=mx, input_len=il)
        add(f"c5/lam{lam}", build_requests(sc, 1), {}, record_tokens=lam != 64)
    g = Xorshift64Star(4242)
    for i in range(30):
        add(f"rand{i}", random_requests(g), random_cost(g), tp=2 if i % 4 == 0 else 1,
            record_tokens=i % 5 != 0)
    _dump("concurrent.json.gz", {"cases": cases}, gz=True)


def gen_suite():
    """suite.py: run_cells -> result_rows -> write_csv on a small grid."""
    from fusionsim import suite as rsuite
    from fusionsim.scenario import ConstantArrival
    sys.path.insert(0, HERE)
    from suite_grid import suite_grid
    grid = suite_grid(Scenario, Discipline, ConstantArrival, PoissonArrival, FixedLength, UniformLength, TPConfig,
                      Placement)
    rsuite.write_csv(rsuite.result_rows(rsuite.run_cells(grid)), os.path.join(HERE, "suite.csv"))


if __name__ == "__main__":
    if len(sys.argv) > 1:
        globals()["gen_" + sys.argv[1]]()
        sys.exit(0)
    gen_suite()
    gen_concurrent()
    gen_dynbatch()
    gen_rng()
    gen_alg1()
    gen_plans()
    gen_requests()
    gen_schedules()
