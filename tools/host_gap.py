"""Host gap per fused iteration under the device clock (each step's duration
is read back before the next boundary): wall time vs summed device time.

    python tools/host_gap.py [--rows 320] [--iters 200]
"""
import argparse, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2305_13484_b200 as fl
from paper_2305_13484_b200.executor import CudaExecutor
from paper_2305_13484_b200.models import get_spec
import bench

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="c3")
ap.add_argument("--rows", type=int, default=320)
ap.add_argument("--iters", type=int, default=200)
a = ap.parse_args()
cfg = bench.CONFIGS[a.config]
spec = get_spec(cfg["spec"])
reqs = [fl.Request(i, 1, cfg["input_len"], cfg["max_out"], cfg["max_out"], 0.0) for i in range(a.rows)]
prompts = fl.synthetic_prompts(reqs, spec.vocab, 1)
ex = CudaExecutor(spec, prompts, dtype=cfg["dtype"], pool_slots=max(a.rows, 8), input_len=cfg["input_len"],
                  max_new_tokens=cfg["max_out"], state_slots=1024, max_rows=max(a.rows, 8) + 256)
st = fl.FusionStream(reqs, fl.CostParams(preprocess_ms=0.0), fl.TPConfig(), executor=ex, record_tokens=False,
                     clock="device")
torch.cuda.set_stream(ex.cs)
st.try_fuse_pending()
for _ in range(20):
    st.step_iteration()
torch.cuda.synchronize()
now0 = st.now
t0 = time.perf_counter()
for _ in range(a.iters):
    st.step_iteration()
torch.cuda.synchronize()
wall = (time.perf_counter() - t0) * 1e3
dev = st.now - now0
print(f"rows={a.rows}: wall {wall / a.iters:.1f} ms/iter, device {dev / a.iters:.3f} ms/iter, "
      f"host gap {1e3 * (wall - dev) / a.iters:.0f} us/iter ({100 * (wall - dev) / wall:.1f} %)")
