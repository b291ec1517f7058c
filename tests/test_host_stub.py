"""The executor's host path on CPU, against a stub library (tests/stub_device.py).

Nothing is computed; these tests pin what the host hands the C-ABI and how
the drop-in engine schedules around it:
* side-stream prefill: the schedule is still the reference's (cost clock),
  every fused request's prompt is imported from its staging slot into its
  physical slot, and no prompt row reaches the fused steps;
* EOS mode: the stop comes from the device's next-token array -- with every
  token equal to the EOS id, every request stops after its first token and
  the trace is the reference schedule of one-token requests;
* the device clock: durations come from the step events, not the cost model.
"""

import ctypes as C

import pytest

torch = pytest.importorskip("torch")

import paper_2305_13484_b200 as fl  # noqa: E402
from paper_2305_13484_b200.core import Request  # noqa: E402
from paper_2305_13484_b200.executor import CudaExecutor  # noqa: E402
from paper_2305_13484_b200.models import get_spec  # noqa: E402
from schedule_dump import load, sha  # noqa: E402
from stub_device import stub_device  # noqa: E402

GOLD = {c["name"]: c for c in load("schedules.json.gz")["cases"]}


def _c1():
    sc = fl.Scenario("t", fl.Discipline.FUSION, 32, fl.PoissonArrival(20.0), fl.UniformLength(8, 64), 64,
                     input_len=16)
    return fl.build_requests(sc, 1)


def _executor(reqs, **kw):
    spec = get_spec("tiny")
    prompts = fl.synthetic_prompts(reqs, spec.vocab, 1)
    return CudaExecutor(spec, prompts, dtype="f32", pool_slots=len(reqs), input_len=16, max_new_tokens=64,
                        state_slots=64, device="cpu", **kw)


@pytest.mark.parametrize("shuffle", [True, False])
def test_side_prefill_host_path(shuffle):
    reqs = _c1()
    with stub_device() as rec:
        ex = _executor(reqs, prefill="side", prefill_slots=8)
        imports = []
        real = ex.lib.fl_step_import

        def spy(h, src, q, s, moves, n):
            imports.extend(tuple(moves[3 * i + j] for j in range(3)) for i in range(n))
            return real(h, src, q, s, moves, n)
        ex.lib.__dict__["fl_step_import"] = spy
        trace = fl.run_fusion(reqs, fl.CostParams(), shuffle_enabled=shuffle, executor=ex)
    assert sha(trace.format_lines()) == GOLD[f"c1/tp1/{'on' if shuffle else 'off'}"]["trace_sha"]
    assert len(imports) == len(reqs)                       # every prompt was staged and imported
    assert all(q < 8 and n == 15 for q, _, n in imports)   # staging slot, P - 1 positions
    assert ex.prefill_rows_total == 0 and ex.lane.passes > 0
    # the lane's own fl_step calls carry only PREFILL rows (n_dec = 0)
    lane_steps = [s for s in rec.steps if s[1] == 0]
    assert len(lane_steps) == ex.lane.passes


def test_eos_mode_host_path():
    reqs = _c1()
    with stub_device():
        ex = _executor(reqs, eos_token=0)          # the stub never writes req_tok: every token is 0
        trace = fl.run_fusion(reqs, fl.CostParams(), executor=ex)
    one = [Request(r.request_id, r.batch_size, r.input_len, r.max_output_length, 1, r.arrival_time)
           for r in reqs]
    assert trace.format_lines() == fl.run_fusion(one, fl.CostParams()).format_lines()


def test_device_clock_uses_step_events():
    reqs = _c1()[:8]
    with stub_device(rank=0):
        ex = _executor(reqs)
        st = fl.FusionStream(reqs, fl.CostParams(preprocess_ms=0.0), fl.TPConfig(), executor=ex,
                             clock="device")
        fl.drive(st)
    # stub events report 1.0 + 0.01 * (k % 7) ms: every iteration lasted ~1 ms
    assert st.device_ms and all(1.0 <= ms < 1.1 for ms in st.device_ms)
    assert len(st.device_ms) == st.iteration_index


def test_tp_mismatch_raises_under_device_clock():
    reqs = _c1()[:4]
    with stub_device():
        ex = _executor(reqs)
        with pytest.raises(fl.InvalidParam):
            fl.FusionStream(reqs, fl.CostParams(), fl.TPConfig(tp_size=2), executor=ex, clock="device")
