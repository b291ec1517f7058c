"""Per-CTA timeline of one k_gemm_sk launch inside a chain of 28 (cold
weights, as the step runs them): dumps the in-kernel debug counters of the
LAST launch to gpurun_out/cta_dump_<M>.json for offline analysis.
    python tools/gemm_cta_dump.py M [M ...]      (ONLY=in|out)"""
import ctypes as C
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

from paper_2305_13484_b200 import _lib  # noqa: E402

lib = _lib.load()
lib.fl_gemm_set_rearm(0)
ws = torch.empty(lib.fl_gemm_workspace_bytes(), dtype=torch.uint8, device="cuda")
L, d, F = 28, 4096, 16384
q3 = 3 * d
only = os.environ.get("ONLY", "in")
N, K = (q3 + F, d) if only == "in" else (d, d + F)


def tile(w):
    n, k = w.shape
    t = torch.empty(lib.fl_tiled_weight_bytes(n, k) // 2, dtype=torch.bfloat16, device="cuda")
    _lib.check(lib.fl_tile_weight(C.c_void_p(w.data_ptr()), n, k, C.c_void_p(t.data_ptr()), None))
    return t


W = [tile((torch.randn(N, K, device="cuda") * 0.02).bfloat16()) for _ in range(L)]
torch.cuda.synchronize()
for M in [int(a) for a in sys.argv[1:]] or [128]:
    h = torch.randn(M, d, device="cuda").bfloat16()
    act = torch.randn(M, 4 * d + F, device="cuda").bfloat16()
    x = torch.zeros(M, d, device="cuda")
    s = torch.cuda.current_stream().cuda_stream

    def one(l):
        if only == "in":
            _lib.check(lib.fl_gemm2(h.data_ptr(), h.data_ptr(), d, W[l].data_ptr(), None, act.data_ptr(), 4 * d + F,
                                    M, N, K, 1, 1, 2, q3, d, None, 0, ws.data_ptr(), C.c_void_p(s)))
        else:
            _lib.check(lib.fl_gemm2(act[:, q3:].data_ptr(), None, 4 * d + F, W[l].data_ptr(), None, x.data_ptr(), d,
                                    M, N, K, 2, 1, 2, 0, 0, None, 0, ws.data_ptr(), C.c_void_p(s)))
    for l in range(L):
        one(l)
    torch.cuda.synchronize()
    dbg = torch.zeros(4 * 8192, dtype=torch.int64, device="cuda")
    for l in range(L - 1):
        one(l)
    lib.fl_gemm_debug(C.c_void_p(dbg.data_ptr()))
    one(L - 1)
    lib.fl_gemm_debug(None)
    torch.cuda.synchronize()
    dd = dbg.view(-1, 4).cpu().tolist()
    os.makedirs("gpurun_out", exist_ok=True)
    json.dump({"M": M, "only": only, "rows": dd[:8192]}, open(f"gpurun_out/cta_dump_{only}_{M}.json", "w"))
    print("dumped", M)
