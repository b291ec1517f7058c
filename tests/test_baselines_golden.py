"""Dynamic batching (C5's comparison discipline) against traces produced by
the reference's run_dynamic_batching (baselines.py:51-127, fixtures from
tests/golden/gen_golden.py)."""

import pytest

import paper_2305_13484_b200 as fl
from schedule_dump import decode_cost, decode_requests, load, sha

CASES = load("dynbatch.json.gz")["cases"]


@pytest.mark.parametrize("case", CASES, ids=[c["name"] for c in CASES])
def test_dynamic_batching_trace_matches_reference(case):
    reqs = [fl.Request(*r) for r in decode_requests(case["requests"])]
    tr = fl.run_dynamic_batching(reqs, fl.BatchWindowConfig(case["window"], case["max_batch"]),
                                 fl.CostParams(**decode_cost(case["cost"])),
                                 fl.TPConfig(tp_size=case["tp"]),
                                 record_tokens=case["record_tokens"]).format_lines()
    assert tr[:len(case["trace_head"])] == case["trace_head"]
    assert len(tr) == case["n_events"]
    assert sha(tr) == case["trace_sha"]


def test_scenario_dispatch_and_fusion_wins():
    sc = fl.Scenario("x", fl.Discipline.DYNAMIC_BATCHING, 24, fl.PoissonArrival(30.0),
                     fl.UniformLength(10, 80), 80, window_ms=50.0)
    db = fl.compute_metrics(fl.run_scenario(sc, 2), 24)
    fu = fl.compute_metrics(fl.run_scenario(
        fl.Scenario("x", fl.Discipline.FUSION, 24, fl.PoissonArrival(30.0),
                    fl.UniformLength(10, 80), 80), 2), 24)
    assert fu.makespan_ms < db.makespan_ms
    with pytest.raises(fl.InvalidParam):
        fl.BatchWindowConfig(-1.0)


CONC = load("concurrent.json.gz")["cases"]


@pytest.mark.parametrize("case", CONC, ids=[c["name"] for c in CONC])
def test_concurrent_instances_trace_matches_reference(case):
    """run_concurrent_instances against traces produced by the
    reference's run_concurrent_instances (baselines.py:130-229)."""
    reqs = [fl.Request(*r) for r in decode_requests(case["requests"])]
    tr = fl.run_concurrent_instances(reqs, fl.CostParams(**decode_cost(case["cost"])),
                                     fl.TPConfig(tp_size=case["tp"]),
                                     record_tokens=case["record_tokens"]).format_lines()
    assert tr[:len(case["trace_head"])] == case["trace_head"]
    assert len(tr) == case["n_events"]
    assert sha(tr) == case["trace_sha"]


def test_concurrent_scenario_dispatch():
    sc = fl.Scenario("x", fl.Discipline.CONCURRENT, 12, fl.PoissonArrival(30.0),
                     fl.UniformLength(10, 40), 40)
    conc = fl.compute_metrics(fl.run_scenario(sc, 3), 12)
    fu = fl.compute_metrics(fl.run_scenario(
        fl.Scenario("x", fl.Discipline.FUSION, 12, fl.PoissonArrival(30.0),
                    fl.UniformLength(10, 40), 40), 3), 12)
    assert conc.makespan_ms > 0 and fu.makespan_ms > 0
    # the device clock needs an executor (device-clock instances: tests/test_gpu_parity.py)
    with pytest.raises(fl.InvalidParam):
        fl.run_scenario(sc, 3, clock="device")
