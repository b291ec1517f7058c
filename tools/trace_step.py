"""Kernel timeline of steady-state fused iterations from CUPTI (torch.profiler).

    python tools/trace_step.py [--config c3] [--rows 128] [--pre 100] [--iters 5]

Unlike the event-bracketed profile (ex.profile), CUPTI's activity records keep
the PDL overlap of the graph: every kernel's own [start, end] on the GPU.
Prints per kernel class: launches per iteration, mean duration, the share of
the iteration's span during which the class runs, and the exposed gaps.
"""
import argparse
import collections
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
from torch.profiler import ProfilerActivity, profile  # noqa: E402

import bench  # noqa: E402
import paper_2305_13484_b200 as fl  # noqa: E402
from paper_2305_13484_b200.executor import CudaExecutor  # noqa: E402
from paper_2305_13484_b200.models import get_spec  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="c3")
ap.add_argument("--rows", type=int, default=128)
ap.add_argument("--pre", type=int, default=100)
ap.add_argument("--iters", type=int, default=5)
ap.add_argument("--json", default=None, help="write the per-class summary here")
a = ap.parse_args()
cfg = bench.CONFIGS[a.config]
spec = get_spec(cfg["spec"])
reqs = [fl.Request(i, 1, cfg["input_len"], cfg["max_out"], cfg["max_out"], 0.0) for i in range(a.rows)]
prompts = fl.synthetic_prompts(reqs, spec.vocab, 1)
ex = CudaExecutor(spec, prompts, dtype=cfg["dtype"], pool_slots=max(a.rows, 8), input_len=cfg["input_len"],
                  max_new_tokens=cfg["max_out"], state_slots=1024, max_rows=max(a.rows, 8) + 256)
st = fl.FusionStream(reqs, fl.CostParams(preprocess_ms=0.0), fl.TPConfig(), executor=ex, record_tokens=False)
torch.cuda.set_stream(ex.cs)
st.try_fuse_pending()
st.step_iteration()
for _ in range(a.pre):
    st.step_iteration()
torch.cuda.synchronize()
with profile(activities=[ProfilerActivity.CUDA]) as prof:
    for _ in range(a.iters):
        st.step_iteration()
    torch.cuda.synchronize()


def klass(name):
    for key, c in (("k_gemm_sk", "gemm"), ("k_attn", "attention"), ("rope", "rope_append"), ("layernorm", "layernorm"),
                   ("k_shuffle", "shuffle"), ("embed", "embed"), ("row_order", "row_order"), ("apply_tokens", "apply"),
                   ("argmax", "argmax")):
        if key in name:
            return c
    return "other:" + name[:40]


ev = []
for e in prof.events():
    if e.device_type == torch.autograd.DeviceType.CUDA and e.time_range.elapsed_us() > 0:
        ev.append((e.time_range.start, e.time_range.end, klass(e.name)))
ev.sort()
if not ev:
    sys.exit("no CUDA kernel records (CUPTI unavailable?)")
span = ev[-1][1] - ev[0][0]
by = collections.defaultdict(lambda: [0, 0.0])
for s, e, c in ev:
    by[c][0] += 1
    by[c][1] += e - s
# busy union and per-class exclusive time over a sweep of the intervals
pts = sorted([(s, 1, c) for s, e, c in ev] + [(e, -1, c) for s, e, c in ev])
active = collections.Counter()
excl = collections.Counter()
busy = 0.0
last = pts[0][0]
for t, d, c in pts:
    n = sum(active.values())
    if n:
        busy += t - last
        if len([k for k, v in active.items() if v]) == 1:
            excl[next(k for k, v in active.items() if v)] += t - last
    active[c] += d
    last = t
it = a.iters
print(f"{a.config} rows={a.rows}: {len(ev) / it:.0f} kernels/iter, span {span / it:.1f} us/iter, "
      f"GPU busy {100 * busy / span:.1f}%")
out = {"config": a.config, "rows": a.rows, "span_us_per_iter": span / it, "busy_pct": 100 * busy / span, "classes": {}}
for c, (n, tot) in sorted(by.items(), key=lambda x: -x[1][1]):
    print(f"  {c:12s} {n / it:6.1f}/iter  mean {tot / n:8.2f} us  sum {tot / it:9.1f} us/iter ({100 * tot / span:5.1f}%)"
          f"  alone {excl[c] / it:9.1f} us/iter ({100 * excl[c] / span:5.1f}%)")
    out["classes"][c] = {"per_iter": n / it, "mean_us": tot / n, "sum_us_per_iter": tot / it,
                         "exclusive_us_per_iter": excl[c] / it}
if a.json:
    json.dump(out, open(a.json, "w"), indent=1)
