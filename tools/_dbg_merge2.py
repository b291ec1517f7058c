import os, sys
sys.path.insert(0, '.'); sys.path.insert(0, 'tests')
import numpy as np, torch
import paper_2305_13484_b200 as fl
from paper_2305_13484_b200.executor import CudaExecutor
from paper_2305_13484_b200.models import get_spec, init_weights
spec = get_spec(sys.argv[1] if len(sys.argv) > 1 else "gptj-mini")
reqs = [fl.Request(i, 1, 16, 8, 8, 0.0) for i in range(int(sys.argv[2]) if len(sys.argv) > 2 else 4)]
prompts = fl.synthetic_prompts(reqs, spec.vocab, 1)
w = init_weights(spec, seed=0, device="cuda", dtype=torch.bfloat16)
out = {}
for mode in ("sep", "merged"):
    if mode == "sep": os.environ["FL_NO_MERGED_OUT"] = "1"
    else: os.environ.pop("FL_NO_MERGED_OUT", None)
    ex = CudaExecutor(spec, prompts, dtype="bf16", pool_slots=8, input_len=16, max_new_tokens=8, state_slots=64,
                      weights=w, capture_logits=True)
    st = fl.FusionStream(reqs, fl.CostParams(preprocess_ms=0.0), fl.TPConfig(), executor=ex)
    fl.drive(st)
    out[mode] = ex.logits_log
    ex.close()
a, b = out["sep"], out["merged"]
print(len(a), len(b))
for i in range(min(len(a), len(b))):
    la, lb = a[i][3], b[i][3]
    print(i, a[i][0], float((la.float() - lb.float()).abs().max()))
