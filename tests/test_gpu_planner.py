"""Device-resident Alg. 1 + plan_shuffle (csrc/planner.cu) against the
reference's golden vectors (tests/golden/alg1.json, plans.json -- generated
by running the reference) and the host planner on random layouts: bit-exact."""

import random

import pytest

torch = pytest.importorskip("torch")

pytestmark = pytest.mark.gpu

import paper_2305_13484_b200 as fl  # noqa: E402
from paper_2305_13484_b200 import devplan  # noqa: E402
from schedule_dump import load  # noqa: E402


def _layout(sizes, evicted, trim=True):
    lay = fl.BufferLayout()
    for rid, size in enumerate(sizes):
        lay.fuse_request(rid, size)
    for rid in evicted:
        lay.evict_request(rid)
    if trim:
        lay.trim_boundaries()
    return lay


def test_device_alg1_matches_reference_golden():
    cases = load("alg1.json")["cases"]
    for arr, off, _cost in cases:
        if not arr:
            continue
        # BufferLayout sizes must be positive: a zero entry is a hole
        sizes = [v if v else 1 for v in arr]
        lay = _layout(sizes, [i for i, v in enumerate(arr) if not v], trim=False)
        assert lay.size_array() == list(arr)
        plan = devplan.device_plan_shuffle(lay)
        assert plan.window_offset - lay.buffer_offset == off, arr


def test_device_plans_match_reference_golden():
    for c in load("plans.json")["cases"]:
        lay = _layout(c["sizes"], c["evicted"])
        plan = devplan.device_plan_shuffle(lay)
        assert [[m.request_id, m.src_slot, m.dst_slot, m.size] for m in plan.moves] == c["moves"]
        assert [plan.window_offset, plan.window_len] == c["plan_window"]
        assert plan.total_bytes_moved == c["bytes"]
        assert plan == fl.plan_shuffle(lay)


@pytest.mark.parametrize("n", [1, 7, 64, 353, 1024, 1025, 4096, 8192])
def test_device_plan_matches_host_random(n):
    rng = random.Random(n)
    for trial in range(4):
        sizes = [rng.choice([1, 3, 1 << 20, rng.randint(1, 1 << 30)]) for _ in range(n)]
        p = rng.random()
        evicted = [i for i in range(n) if rng.random() < p and i not in (0, n - 1)]
        lay = _layout(sizes, evicted)
        assert devplan.device_plan_shuffle(lay) == fl.plan_shuffle(lay), (n, trial)


def test_device_plan_rejects_oversized_window():
    lay = _layout([1] * 8193, [])
    with pytest.raises(ValueError):
        devplan.device_plan_shuffle(lay)


@pytest.mark.parametrize("shuffle_seed", [1, 7])
def test_device_planner_in_the_serving_loop(monkeypatch, shuffle_seed):
    """every shuffle boundary planned AND executed on the device
    (fl_shuffle_planned: Alg. 1 + plan_shuffle in csrc/planner.cu, K10 fed
    from the device move list).  The host planner is taken out of the loop
    (it raises if called), yet the trace is the reference's golden trace and
    the tokens equal the host-planned run's and the oracle's."""
    from harness import oracle_check, run_device, scenario_requests
    from schedule_dump import sha
    import paper_2305_13484_b200.engine as eng
    gold = {c["name"]: c for c in load("schedules.json.gz")["cases"]}["c1/tp1/on"]
    reqs = scenario_requests(32, 20.0, 8, 64, 64, 16, seed=shuffle_seed)
    _, _, host, _, _ = run_device("tiny", reqs, dtype="f32", shuffle=True, capture_logits=False)

    def no_host_plan(*a, **k):
        raise AssertionError("host plan_shuffle called in device-plan mode")
    monkeypatch.setattr(eng, "plan_shuffle", no_host_plan)
    trace, st, ex, prompts, w32 = run_device("tiny", reqs, dtype="f32", shuffle=True, device_plan=True)
    if shuffle_seed == 1:
        assert sha(trace.format_lines()) == gold["trace_sha"]
    assert ex.device_plans > 0 and ex.shuffles == host.shuffles > 0
    assert ex.moved_kv_bytes == host.moved_kv_bytes
    assert ex.tokens() == host.tokens()
    stats = oracle_check("tiny", ex, prompts, w32, logit_atol=2e-3, logit_rtol=1e-3, margin=5e-3)
    assert stats["mismatched"] == 0, stats


def test_device_planner_device_clock_bf16():
    """Device clock + tcgen05 path: the measured shuffle time covers planner
    + K10; all requests complete with their full token counts."""
    from harness import run_device, scenario_requests
    reqs = scenario_requests(32, 0.1, 4, 40, 40, 16, seed=3)      # all live at once: holes
    trace, st, ex, _, _ = run_device("gptj-mini", reqs, dtype="bf16", shuffle=True, device_plan=True,
                                     clock="device", params=fl.CostParams(preprocess_ms=0.0),
                                     capture_logits=False)
    assert ex.device_plans > 0
    assert all(ms > 0 for _, _, ms in ex.shuffle_log)
    toks = ex.tokens()
    assert [len(toks[r.request_id]) for r in reqs] == [r.actual_output_length for r in reqs]


@pytest.mark.parametrize("shuffle", [True, False])
def test_eos_token_stop(shuffle):
    """Data-dependent EOS: requests stop at their first greedy
    EOS token instead of a pre-sampled length.  Bars: each stream is the
    prefix (through the first EOS) of the same request's stream run to
    max_output_length; and the device run's trace equals the reference
    schedule of requests whose actual_output_length is the discovered stop
    (record_token's eos_at, reference core.py:108-123) -- bit-exact."""
    from collections import Counter
    from harness import run_device, scenario_requests
    from paper_2305_13484_b200.core import Request
    reqs = scenario_requests(24, 10.0, 40, 40, 40, 16, seed=9)      # every request runs to 40
    _, _, full, _, _ = run_device("tiny", reqs, dtype="f32", shuffle=shuffle, capture_logits=False)
    ftok = full.tokens()
    # the EOS token: the most frequent token in the first halves of the streams
    eos = Counter(t for v in ftok.values() for t in v[:20]).most_common(1)[0][0]
    trace, st, ex, _, _ = run_device("tiny", reqs, dtype="f32", shuffle=shuffle, capture_logits=False,
                                     executor_opts=dict(eos_token=eos))
    toks = ex.tokens()
    stops = {}
    for r in reqs:
        f = ftok[r.request_id]
        k = f.index(eos) + 1 if eos in f else len(f)
        stops[r.request_id] = k
        assert toks[r.request_id] == f[:k], r.request_id
    assert any(k < 40 for k in stops.values())
    ref = [Request(r.request_id, r.batch_size, r.input_len, r.max_output_length, stops[r.request_id],
                   r.arrival_time) for r in reqs]
    expect = fl.run_fusion(ref, fl.CostParams(), shuffle_enabled=shuffle)
    assert trace.format_lines() == expect.format_lines()
