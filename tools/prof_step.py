"""Steady-state fused-iteration probe: host time per fl_step vs device time.

    python tools/prof_step.py [--config c2] [--rows 48] [--iters 200]

Builds the config's executor, fuses `rows` requests at once, runs `iters`
iterations (cost clock, no per-step sync) and reports host launch time per
iteration, device time per iteration (CUDA events), and per-class kernel time.
"""
import argparse, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2305_13484_b200 as fl
from paper_2305_13484_b200.executor import CudaExecutor
from paper_2305_13484_b200.models import get_spec
import bench

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="c2")
ap.add_argument("--rows", type=int, default=48)
ap.add_argument("--iters", type=int, default=200)
ap.add_argument("--profile", action="store_true")
ap.add_argument("--pre", type=int, default=5, help="decode iterations before the measured loop (context growth)")
ap.add_argument("--dump", default=None, help="with --profile: write per-class algorithmic bytes/launch JSON here")
a = ap.parse_args()
cfg = bench.CONFIGS[a.config]
spec = get_spec(cfg["spec"])
reqs = [fl.Request(i, 1, cfg["input_len"], cfg["max_out"], cfg["max_out"], 0.0) for i in range(a.rows)]
prompts = fl.synthetic_prompts(reqs, spec.vocab, 1)
ex = CudaExecutor(spec, prompts, dtype=cfg["dtype"], pool_slots=max(a.rows, 8), input_len=cfg["input_len"],
                  max_new_tokens=cfg["max_out"], state_slots=1024, max_rows=max(a.rows, 8) + 256)
# TUNE="7=1,...": fl_gemm_tune diagnostics for every graph this run captures (results garbage, timing valid)
for kv in filter(None, (os.environ.get("TUNE") or "").split(",")):
    k, v = kv.split("=")
    ex.lib.fl_gemm_tune(int(k), int(v))
st = fl.FusionStream(reqs, fl.CostParams(preprocess_ms=0.0), fl.TPConfig(), executor=ex, record_tokens=False)
torch.cuda.set_stream(ex.cs)
st.try_fuse_pending()
st.step_iteration()            # admission step (prefill rows)
for _ in range(a.pre):
    st.step_iteration()
torch.cuda.synchronize()
if a.profile:
    ex.profile(True)
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
torch.cuda.profiler.start()          # ncu --profile-from-start off: steady-state decode only
e0.record()
t0 = time.perf_counter()
for _ in range(a.iters):
    st.step_iteration()
t1 = time.perf_counter()
e1.record(); torch.cuda.synchronize()
torch.cuda.profiler.stop()
t2 = time.perf_counter()
print(f"rows={a.rows} host launch {1e6*(t1-t0)/a.iters:.1f} us/iter, wall {1e6*(t2-t0)/a.iters:.1f} us/iter, "
      f"device {1e3*e0.elapsed_time(e1)/a.iters:.1f} us/iter")
if a.profile:
    pr = ex.profile_read()
    for k, v in pr.items():
        print(k, f"{1e3*v['ms']/a.iters:.1f} us/iter", v["records"], "records")
    if a.dump:
        import json
        att_b = ex.attn_bytes_profiled
        out = {"rows": a.rows, "config": a.config, "pre": a.pre}
        for k, v in pr.items():
            if v["records"]:
                b = att_b if k == "attention" else v["bytes"]
                out[k] = {"algorithmic_bytes_per_launch": b / v["records"], "records": v["records"],
                          "us_per_launch": 1e3 * v["ms"] / v["records"]}
        json.dump(out, open(a.dump, "w"), indent=1)
