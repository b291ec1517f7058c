"""Back-to-back projection GEMM timing (CUDA graph of repeated launches).

    python tools/gemm_bench.py  -> ours (tcgen05) vs torch/cuBLAS per shape
"""
import ctypes as C
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2305_13484_b200 import _lib

lib = _lib.load()
ws = torch.empty(lib.fl_gemm_workspace_bytes(), dtype=torch.uint8, device="cuda")
REPS = 50
shapes = [(48, 2304, 768), (48, 768, 768), (48, 3072, 768), (48, 768, 3072), (48, 50257, 768),
          (112, 2304, 768), (112, 768, 3072), (1, 768, 3072), (100, 12288, 4096), (100, 4096, 16384)]
if len(sys.argv) > 1:
    shapes = [tuple(map(int, a.split("x"))) for a in sys.argv[1:]]
s = torch.cuda.Stream()
dbg = torch.zeros(4 * 4096, dtype=torch.int64, device="cuda")
for M, N, K in shapes:
    x = torch.randn(M, K, device="cuda").bfloat16()
    w = (torch.randn(N, K, device="cuda") * 0.02).bfloat16()
    out = torch.empty(M, N, device="cuda", dtype=torch.bfloat16)
    def ours():
        _lib.check(lib.fl_gemm(x.data_ptr(), K, w.data_ptr(), None, out.data_ptr(), N, M, N, K, 0, 1, 1,
                               ws.data_ptr(), C.c_void_p(torch.cuda.current_stream().cuda_stream)))
    def ref():
        torch.matmul(x, w.T, out=out)
    res = []
    for name, fn in (("ours", ours), ("torch", ref)):
        with torch.cuda.stream(s):
            fn(); torch.cuda.synchronize()
            g = torch.cuda.CUDAGraph()
            with torch.cuda.graph(g, stream=s):
                for _ in range(REPS):
                    fn()
            g.replay(); torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(s)
            for _ in range(5):
                g.replay()
            e1.record(s); torch.cuda.synchronize()
        us = e0.elapsed_time(e1) * 1e3 / (5 * REPS)
        gbs = (N * K * 2 + M * K * 2 + M * N * 2) / us / 1e3
        res.append(f"{name} {us:7.2f} us {gbs:7.0f} GB/s")
    print(f"M={M:4d} N={N:6d} K={K:6d}  " + "   ".join(res), flush=True)
    if os.environ.get("GEMM_DBG"):
        dbg.zero_(); lib.fl_gemm_debug(C.c_void_p(dbg.data_ptr())); ours(); torch.cuda.synchronize()
        lib.fl_gemm_debug(None)
        d = dbg.view(-1, 4).cpu().double(); d = d[d[:, 3] > 0]
        print(f"   CTAs {len(d)}: producer waits {100*d[:,0].sum()/d[:,1].sum():.0f}% of {d[:,1].mean():.0f} clk, "
              f"mma waits {100*d[:,2].sum()/d[:,3].sum():.0f}% of {d[:,3].mean():.0f} clk")
