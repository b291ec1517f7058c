"""Shared drivers for the GPU parity tests, smoke() and bench.py's checks."""

from __future__ import annotations

import numpy as np

import paper_2305_13484_b200 as fl
from paper_2305_13484_b200.executor import CudaExecutor
from paper_2305_13484_b200.models import get_spec, init_weights


def scenario_requests(n, mean_ms, lo, hi, max_out, input_len, seed=1):
    sc = fl.Scenario("t", fl.Discipline.FUSION, n, fl.PoissonArrival(mean_ms),
                     fl.UniformLength(lo, hi), max_out, input_len=input_len)
    return fl.build_requests(sc, seed)


def run_device(spec_name, requests, *, dtype="f32", shuffle=True, clock="cost", seed=1,
               params=None, tp=None, capture_logits=True, pool_slots=None, use_tc=None,
               weights=None, record_tokens=True, time_steps=False, comm_id=None, device_plan=False,
               executor_opts=None):
    """Serve ``requests`` through the drop-in engine on the device.
    Returns (trace, stream, executor, prompts, weights_cpu_fp32)."""
    import torch
    spec = get_spec(spec_name)
    prompts = fl.synthetic_prompts(requests, spec.vocab, seed)
    max_out = max(r.max_output_length for r in requests)
    input_len = max(r.input_len for r in requests)
    tdt = torch.float32 if dtype == "f32" else torch.bfloat16
    if weights is None:
        weights = init_weights(spec, seed=0, device="cuda", dtype=tdt)
    ex = CudaExecutor(spec, prompts, dtype=dtype, pool_slots=pool_slots or len(requests),
                      max_new_tokens=max_out, input_len=input_len,
                      state_slots=max(64, len(requests)), weights=weights,
                      use_tensor_cores=use_tc, capture_logits=capture_logits,
                      time_steps=time_steps, comm_id=comm_id, device_plan=device_plan,
                      **(executor_opts or {}))
    st = fl.FusionStream(requests, params or fl.CostParams(), tp or fl.TPConfig(),
                         shuffle_enabled=shuffle, record_tokens=record_tokens, executor=ex,
                         clock=clock)
    fl.drive(st)
    trace = fl.Trace("fusion" if shuffle else "fusion_noshuffle", st.events)
    trace.sort()
    w32 = {k: v.float().cpu().numpy() for k, v in weights.items()}
    return trace, st, ex, prompts, w32


def oracle_check(spec_name, ex, prompts, w32, *, logit_atol, logit_rtol, margin):
    """Teacher-forced oracle replay; returns stats and asserts nothing."""
    from oracle.model_oracle import GPTOracle, replay
    spec = get_spec(spec_name)
    orc = GPTOracle.from_spec(spec, w32, ex.S)
    toks = ex.tokens()
    worst = 0.0
    n = exact = ambiguous = mismatched = 0
    for it, rid, c, lo, ld, tok in replay(orc, ex.logits_log, prompts, toks):
        err = np.abs(lo - ld[:spec.vocab]) - logit_rtol * np.abs(lo)
        worst = max(worst, float(err.max()))
        n += 1
        top = int(np.argmax(lo))
        srt = np.sort(lo)
        gap = float(srt[-1] - srt[-2])
        if tok == top:
            exact += 1
        elif gap < margin or lo[tok] >= lo[top] - margin:
            ambiguous += 1
        else:
            mismatched += 1
    return {"rows": n, "exact": exact, "ambiguous": ambiguous, "mismatched": mismatched,
            "worst_excess": worst, "atol": logit_atol}
