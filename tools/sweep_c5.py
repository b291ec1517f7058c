"""C5: arrival-rate sweep on the GPT-J 6B shape -- temporal fusion vs dynamic
batching, both executed on the B200 with the device clock.

    python tools/sweep_c5.py [--n 64] [--rates 1,2,4,8,16,32,64] [--window 50]

For each rate lambda (req/s) the same request stream (reference generator,
PoissonArrival(1000/lambda), U(128,1024) outputs) is served by
(a) the fused stream (shuffle on, admission control at the pool size) and
(b) dynamic batching with a fixed batch window (reference baselines.py:51-127),
and we report decode tokens/s over device-busy time, makespan and p50/p99
request latency (evicted - arrived, device clock).  One JSON line per rate.
"""

import argparse
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch

import paper_2305_13484_b200 as fl
from paper_2305_13484_b200.executor import CudaExecutor
from paper_2305_13484_b200.models import get_spec


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=64)
    ap.add_argument("--rates", default="1,2,4,8,16,32,64")
    ap.add_argument("--window", type=float, default=50.0)
    ap.add_argument("--spec", default="gptj-6b")
    ap.add_argument("--seed", type=int, default=1)
    ap.add_argument("--instances-max-rate", type=float, default=0.0,
                    help="also run concurrent instances (device clock, one batch-1 decoder per live request on "
                         "its own stream) at rates up to this many req/s")
    a = ap.parse_args()
    spec = get_spec(a.spec)
    params = fl.CostParams(preprocess_ms=0.0)
    ex = None
    for lam in [float(x) for x in a.rates.split(",")]:
        sc = fl.Scenario("c5", fl.Discipline.FUSION, a.n, fl.PoissonArrival(1000.0 / lam),
                         fl.UniformLength(128, 1024), 1024, input_len=32)
        reqs = fl.build_requests(sc, a.seed)
        prompts = fl.synthetic_prompts(reqs, spec.vocab, a.seed)
        if ex is None:
            ex = CudaExecutor(spec, prompts, dtype="bf16", pool_slots=0, input_len=32,
                              max_new_tokens=1024, state_slots=max(64, a.n))
            torch.cuda.set_stream(ex.cs)
        ex.prompts = prompts
        tokens = sum(r.actual_output_length for r in reqs)
        out = {"lambda_req_s": lam, "requests": a.n, "tokens": tokens, "model": a.spec}
        names = ["fusion", "dynamic_batching"]
        if lam <= a.instances_max_rate:
            names.append("concurrent_instances")
        for name in names:
            ex.reset()
            t0 = time.perf_counter()
            if name == "fusion":
                st = fl.FusionStream(reqs, params, fl.TPConfig(), executor=ex, clock="device",
                                     max_window=ex.C)
                fl.drive(st)
                tr = fl.Trace("fusion", st.events)
                tr.sort()
                busy = sum(st.device_ms)
            elif name == "dynamic_batching":
                tr = fl.run_dynamic_batching(reqs, fl.BatchWindowConfig(a.window), params,
                                             executor=ex, clock="device")
                busy = sum(e.value for e in tr.of_kind(fl.EventKind.ITERATION_COMPLETED))
            else:
                tr = fl.run_concurrent_instances(reqs, params, executor=ex, clock="device",
                                                 max_instances=64)
                m0 = fl.compute_metrics(tr, a.n)
                busy = m0.makespan_ms              # instances overlap: device time = their span
            wall = time.perf_counter() - t0
            m = fl.compute_metrics(tr, a.n)
            out[name] = {"tokens_per_s_busy": tokens / (busy / 1e3), "busy_ms": busy,
                         "makespan_ms": m.makespan_ms, "p50_ms": m.p50_latency_ms,
                         "p99_ms": m.p99_latency_ms, "iterations": m.total_stream_iterations,
                         "wall_s": wall}
        out["fusion_speedup_makespan"] = (out["dynamic_batching"]["makespan_ms"]
                                          / out["fusion"]["makespan_ms"])
        out["fusion_speedup_p50"] = out["dynamic_batching"]["p50_ms"] / out["fusion"]["p50_ms"]
        print(json.dumps(out), flush=True)


if __name__ == "__main__":
    main()
