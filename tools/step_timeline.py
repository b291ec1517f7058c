"""In-kernel %globaltimer timeline of the LAST layer of one fused iteration:
attention (fl_attention_debug) then the out-projection GEMM and the LM head
(fl_gemm_debug, alternating halves) -- when each kernel's CTAs start, when
their grid dependency resolves and when they end.

    python tools/step_timeline.py [--config c3] [--rows 128] [--pre 100]
"""
import argparse
import ctypes as C
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import bench  # noqa: E402
import paper_2305_13484_b200 as fl  # noqa: E402
from paper_2305_13484_b200.executor import CudaExecutor  # noqa: E402
from paper_2305_13484_b200.models import get_spec  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="c3")
ap.add_argument("--rows", type=int, default=128)
ap.add_argument("--pre", type=int, default=100)
a = ap.parse_args()
cfg = bench.CONFIGS[a.config]
spec = get_spec(cfg["spec"])
reqs = [fl.Request(i, 1, cfg["input_len"], cfg["max_out"], cfg["max_out"], 0.0) for i in range(a.rows)]
prompts = fl.synthetic_prompts(reqs, spec.vocab, 1)
ex = CudaExecutor(spec, prompts, dtype=cfg["dtype"], pool_slots=max(a.rows, 8), input_len=cfg["input_len"],
                  max_new_tokens=cfg["max_out"], state_slots=1024, max_rows=max(a.rows, 8) + 256)
st = fl.FusionStream(reqs, fl.CostParams(preprocess_ms=0.0), fl.TPConfig(), executor=ex, record_tokens=False)
torch.cuda.set_stream(ex.cs)
# GEMM launches bake the debug pointer into the captured graphs: set both
# before the first step (attention reads its pointer at run time)
lib = ex.lib
gd = torch.zeros(2 * 4 * 16384, dtype=torch.int64, device="cuda")
ad = torch.zeros(64 * 296, dtype=torch.int64, device="cuda")
lib.fl_gemm_tune(9, 1)     # alternate halves: the last two GEMM launches
lib.fl_gemm_debug(C.c_void_p(gd.data_ptr()))
lib.fl_attention_debug(C.c_void_p(ad.data_ptr()))
st.try_fuse_pending()
st.step_iteration()
for _ in range(a.pre):
    st.step_iteration()
torch.cuda.synchronize()
gd.zero_()
ad.zero_()
st.step_iteration()
torch.cuda.synchronize()
lib.fl_gemm_debug(None)
lib.fl_attention_debug(None)

att = ad.view(296, 64).cpu().double()
att = att[att[:, 0] > 0]
rows = []
if len(att):
    ends = []
    for r in att:
        e = [r[3 + 2 * i] for i in range(31) if r[3 + 2 * i] > 0]
        ends.append(max(e) if e else r[1])
    rows.append(("attention", att[:, 0].min(), att[:, 0].max(), att[:, 1].max(), min(ends), max(ends)))
for i in range(2):
    hv = gd[i * 4 * 16384:(i + 1) * 4 * 16384].view(-1, 4).cpu().double()
    ok = (hv[4096:6144, 0] > 0) & (hv[8192:8192 + 2048, 3] > 0)
    if ok.any():
        rows.append((f"gemm half {i}", hv[4096:6144, 0][ok].min(), hv[4096:6144, 0][ok].max(),
                     hv[8192:8192 + 2048, 0][ok].max(), hv[8192:8192 + 2048, 3][ok].min(),
                     hv[8192:8192 + 2048, 3][ok].max()))
if not rows:
    sys.exit("no stamps (graphs replayed without the debug pointers?)")
rows.sort(key=lambda r: r[1])
Z = rows[0][1]
for name, s0, s1, dep, e0, e1 in rows:
    print(f"{name:14s} CTAs start {(s0 - Z) / 1e3:8.2f}..{(s1 - Z) / 1e3:8.2f} us | dependency resolved by"
          f" {(dep - Z) / 1e3:8.2f} | end {(e0 - Z) / 1e3:8.2f}..{(e1 - Z) / 1e3:8.2f}")
