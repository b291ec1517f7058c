"""The product's drop-in host API against the reference's golden vectors and
its own known-answer cases (reference tests/test_engine.py:43-221,
tests/test_buffer.py, tests/prop_helpers.py:126-189)."""

import pytest

import paper_2305_13484_b200 as fl
from paper_2305_13484_b200 import buffer as fb
from schedule_dump import decode_cost, decode_requests, iter_line, load, sha

EK = fl.EventKind


# ------------------------------------------------------------------ rng
def test_rng_matches_reference():
    g = load("rng.json")
    for seed, stream, want in g["derive"]:
        assert fl.rng.derive_seed(seed, stream) == want
    for case in g["streams"]:
        x = fl.rng.Xorshift64Star(case["seed"], case["stream"])
        assert [x.next_u64() for _ in range(16)] == case["u64"]
        assert [x.next_float().hex() for _ in range(8)] == case["float"]
        ints = [x.uniform_int(0, 50256) for _ in range(8)] + [x.uniform_int(128, 1024) for _ in range(8)]
        assert ints == case["int"]
        assert [x.exponential(20.0).hex() for _ in range(8)] == case["exp"]


def test_requests_match_reference():
    g = load("requests.json")
    spec = {"c1": (32, 8, 64, 64, 16), "c2": (128, 32, 512, 512, 32),
            "c3": (512, 128, 1024, 1024, 32), "c4": (64, 128, 1024, 1024, 32)}
    for key, rows in g.items():
        name, seed = key.split("/")
        if name == "const":
            sc = fl.Scenario("k", fl.Discipline.FUSION, 16, fl.ConstantArrival(20.0),
                             fl.UniformLength(128, 1792), 1792)
        else:
            n, lo, hi, mx, il = spec[name]
            sc = fl.Scenario(name, fl.Discipline.FUSION, n, fl.PoissonArrival(20.0),
                             fl.UniformLength(lo, hi), mx, input_len=il)
        got = [[r.request_id, r.batch_size, r.input_len, r.max_output_length,
                r.actual_output_length, r.arrival_time.hex()] for r in fl.build_requests(sc, int(seed))]
        assert got == rows, key


# ------------------------------------------------------------------ Alg.1 / plans
def test_alg1_matches_reference():
    for arr, off, cost in load("alg1.json")["cases"]:
        assert fl.find_shuffled_memory_region(arr) == off
        assert fb.window_move_cost(arr, off) == cost
        if len(arr) <= 64:
            assert fl.brute_force_min_window(arr) == (off, cost)


def test_plans_match_reference():
    for c in load("plans.json")["cases"]:
        lay = fl.BufferLayout()
        for rid, size in enumerate(c["sizes"]):
            lay.fuse_request(rid, size)
        for rid in c["evicted"]:
            lay.evict_request(rid)
        lay.trim_boundaries()
        assert [lay.buffer_offset, lay.buffer_size] == c["window"]
        plan = fl.plan_shuffle(lay)
        assert [[m.request_id, m.src_slot, m.dst_slot, m.size] for m in plan.moves] == c["moves"]
        assert [plan.window_offset, plan.window_len] == c["plan_window"]
        assert plan.total_bytes_moved == c["bytes"]
        fl.apply_shuffle(lay, plan)
        if plan.moves:
            assert not lay.has_interior_holes()


def test_layout_errors():
    lay = fl.BufferLayout(capacity=2)
    lay.fuse_request(0, 10)
    with pytest.raises(fl.DuplicateRequest):
        lay.fuse_request(0, 10)
    lay.fuse_request(1, 30)
    with pytest.raises(fl.CapacityExceeded):
        lay.fuse_request(2, 1)
    with pytest.raises(fl.UnknownRequest):
        lay.evict_request(7)
    lay2 = fl.BufferLayout()
    for rid, s in enumerate([10, 0 + 5, 30]):
        lay2.fuse_request(rid, s)
    lay2.evict_request(0)
    plan = fl.plan_shuffle(lay2)
    lay2.evict_request(1)
    with pytest.raises(fl.StalePlan):
        fl.apply_shuffle(lay2, plan)
    with pytest.raises(fl.OracleBoundExceeded):
        fl.brute_force_min_window([1] * 5000)


def test_exact_plan_and_offsets():
    # reference tests/test_buffer.py:156-179: [10,0,30] -> slot 0 moves to 1
    lay = fl.BufferLayout()
    for rid, s in enumerate([10, 20, 30]):
        lay.fuse_request(rid, s)
    lay.evict_request(1)
    plan = fl.plan_shuffle(lay)
    assert [(m.request_id, m.src_slot, m.dst_slot, m.size) for m in plan.moves] == [(0, 0, 1, 10)]
    fl.apply_shuffle(lay, plan)
    assert lay.per_request_offset == {0: 1, 2: 2}
    assert (lay.buffer_offset, lay.buffer_size) == (1, 2)


# ------------------------------------------------------------------ engine
SCHED = load("schedules.json.gz")["cases"]


def _stream_dump(case, executor=None):
    reqs = [fl.Request(*r) for r in decode_requests(case["requests"])]
    params = fl.CostParams(**decode_cost(case["cost"]))
    tp = fl.TPConfig(case["tp"], fl.Placement(case["placement"]))
    st = fl.FusionStream(reqs, params, tp, shuffle_enabled=case["shuffle"],
                         record_tokens=case["record_tokens"], executor=executor)
    lines = []
    it = 0
    while not st.finished_all():
        if not st.active:
            st.now = max(st.now, st.next_ready_time())
        before = set(st.active)
        st.try_fuse_pending()
        lay = st.layout
        admitted = [[rid, lay.per_request_offset[rid]] for rid in st.active if rid not in before]
        win0 = lay.buffer_offset
        rows = [(-1 if lay.slots[s].occupant is None else lay.slots[s].occupant)
                for s in range(lay.buffer_offset, lay.buffer_offset + lay.buffer_size)]
        offs = dict(lay.per_request_offset)
        t0 = st.now
        n_ev = len(st._ev)
        st.step_iteration()
        new = st._ev[n_ev:]
        fin = [e.request_id for e in new if e.kind is EK.EVICTED]
        dur = [e.value for e in new if e.kind is EK.ITERATION_COMPLETED][0]
        sh = [e.value for e in new if e.kind is EK.SHUFFLE_EXECUTED]
        moves = sorted([[rid, offs[rid], s, lay.slots[s].size]
                        for rid, s in lay.per_request_offset.items() if offs[rid] != s],
                       key=lambda m: m[1])
        lines.append(iter_line(it, t0, dur, win0, rows, admitted, fin, moves,
                               sh[0] if sh else 0, st.now, (lay.buffer_offset, lay.buffer_size)))
        it += 1
        # stepwise layout integrity (prop_helpers.py:143-158)
        assert set(lay.per_request_offset) == set(st.active)
        for rid, idx in lay.per_request_offset.items():
            assert lay.slots[idx].occupant == rid
            assert lay.slots[idx].size == st.active[rid].tensor_size
        if case["shuffle"]:
            assert not lay.has_interior_holes()
    return lines


@pytest.mark.parametrize("case", SCHED, ids=[c["name"] for c in SCHED])
def test_engine_schedule_matches_reference(case):
    lines = _stream_dump(case)
    assert lines[:len(case["iters"])] == case["iters"]
    assert sha(lines) == case["iter_sha"]
    reqs = [fl.Request(*r) for r in decode_requests(case["requests"])]
    params = fl.CostParams(**decode_cost(case["cost"]))
    tp = fl.TPConfig(case["tp"], fl.Placement(case["placement"]))
    trace = fl.run_fusion(reqs, params, tp, shuffle_enabled=case["shuffle"],
                          record_tokens=case["record_tokens"]).format_lines()
    assert trace[:len(case["trace_head"])] == case["trace_head"]
    assert sha(trace) == case["trace_sha"]


TIGHT = fl.CostParams(base_iteration_ms=10.0, marginal_per_request_ms=0.0, preprocess_ms=10.0,
                      alpha_intra_ms=0.0, beta_intra_ms_per_byte=2.0**-10,
                      memcpy_beta_ms_per_byte=2.0**-10, request_bytes=100)


def _req(rid, arrival, n, max_out=None):
    return fl.Request(rid, 1, 32, max_out or n, n, arrival)


def test_known_answers_from_reference_tests():
    # test_engine.py:43-50
    m = fl.compute_metrics(fl.run_fusion([_req(0, 0.0, 512)], fl.CostParams()), 1)
    assert m.makespan_ms == 6011.71875 and m.total_stream_iterations == 512
    # test_engine.py:66-77
    tr = fl.run_fusion([_req(0, 0.0, 5), _req(1, 10.0, 2), _req(2, 15.0, 1)], TIGHT)
    fused = {e.request_id: e.time for e in tr.of_kind(EK.FUSED)}
    assert fused == {0: 10.0, 1: 20.0, 2: 30.0}
    # test_engine.py:113-167 orphan slots at TP=2
    d300 = 10.0 + 3.0 * (150.0 * 2.0**-10)
    d200 = 10.0 + 3.0 * (100.0 * 2.0**-10)
    reqs = [_req(i, 0.0, n) for i, n in enumerate([3, 1, 3])]
    on = fl.run_fusion(reqs, TIGHT, fl.TPConfig(tp_size=2), shuffle_enabled=True)
    assert [e.value for e in on.of_kind(EK.ITERATION_COMPLETED)] == [d300, d200, d200]
    assert [e.value for e in on.of_kind(EK.SHUFFLE_EXECUTED)] == [100]
    off = fl.run_fusion(reqs, TIGHT, fl.TPConfig(tp_size=2), shuffle_enabled=False)
    assert [e.value for e in off.of_kind(EK.ITERATION_COMPLETED)] == [d300] * 3


def test_empty_stream_and_no_requests():
    st = fl.FusionStream([], TIGHT, fl.TPConfig())
    with pytest.raises(fl.EmptyStream):
        st.step_iteration()
    assert fl.run_fusion([], TIGHT).events == []


def test_active_table_view_semantics():
    reqs = [_req(i, 0.0, 3 + i) for i in range(3)]
    st = fl.FusionStream(reqs, TIGHT, fl.TPConfig())
    st.now = st.next_ready_time()
    st.try_fuse_pending()
    assert list(st.active) == [0, 1, 2]
    st.step_iteration()
    assert [st.active[r].current_iteration for r in st.active] == [1, 1, 1]
    assert st.active[1].memory_offset == 1
    info = st.active[2]
    assert isinstance(info, fl.RuntimeInfo) and info.max_output_length == 5


def test_record_token_and_phases():
    info = fl.RuntimeInfo(0, 0, 10, "gpu", 3, 2)
    nxt, done = fl.record_token(info, 5)
    assert nxt.current_iteration == 3 and done
    with pytest.raises(fl.AlreadyFinished):
        fl.record_token(nxt, 5)
    with pytest.raises(fl.InvalidParam):
        fl.record_token(info, 0)
    with pytest.raises(fl.IllegalTransition):
        fl.advance_phase(fl.Phase.RECEIVED, fl.Phase.RUNNING)
    assert fl.Phase.RUNNING.successor() is fl.Phase.FINISHED
    assert fl.Phase.FINISHED.successor() is None


def test_metrics_percentile_convention():
    assert fl.percentile([1.0, 2.0, 3.0, 4.0], 50.0) == 2.5
    assert fl.percentile([5.0], 99.0) == 5.0
    with pytest.raises(fl.InvalidParam):
        fl.percentile([], 50.0)


def test_admission_control_caps_the_window():
    """Extension: max_window keeps contexts queued while the KV pool is full."""
    sc = fl.Scenario("x", fl.Discipline.FUSION, 40, fl.PoissonArrival(2.0), fl.UniformLength(3, 30), 30)
    reqs = fl.build_requests(sc, 3)
    for shuffle in (True, False):
        st = fl.FusionStream(reqs, fl.CostParams(), fl.TPConfig(), shuffle_enabled=shuffle,
                             max_window=5)
        fl.drive(st)
        assert st.widest_window <= 5
        tr = fl.Trace("f", st.events)
        toks = {}
        for e in tr.events:
            if e.kind is EK.TOKEN_GENERATED:
                toks[e.request_id] = toks.get(e.request_id, 0) + 1
        assert toks == {r.request_id: r.actual_output_length for r in reqs}
    # None keeps the reference schedule
    a = fl.run_fusion(reqs, fl.CostParams()).format_lines()
    b = fl.run_fusion(reqs, fl.CostParams(), max_window=None).format_lines()
    assert a == b
