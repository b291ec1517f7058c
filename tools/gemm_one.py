"""Run one projection GEMM shape a few times (no graph) -- for ncu captures.

    python tools/gemm_one.py 320x12288x4096 [epi]
"""
import ctypes as C
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2305_13484_b200 import _lib

lib = _lib.load()
ws = torch.empty(lib.fl_gemm_workspace_bytes(), dtype=torch.uint8, device="cuda")
M, N, K = map(int, sys.argv[1].split("x"))
epi = int(sys.argv[2]) if len(sys.argv) > 2 else 0
x = torch.randn(M, K, device="cuda").bfloat16()
w = (torch.randn(N, K, device="cuda") * 0.02).bfloat16()
out = torch.zeros(M, N, device="cuda", dtype=torch.bfloat16 if epi in (0, 1) else torch.float32)
for _ in range(int(os.environ.get("REPS", "3"))):
    _lib.check(lib.fl_gemm(x.data_ptr(), K, w.data_ptr(), None, out.data_ptr(), N, M, N, K, epi, 1, 1,
                           ws.data_ptr(), C.c_void_p(torch.cuda.current_stream().cuda_stream)))
torch.cuda.synchronize()
print("ok", M, N, K, epi)
