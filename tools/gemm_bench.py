"""Back-to-back projection GEMM timing (CUDA graph of repeated launches).

    python tools/gemm_bench.py  -> ours (tcgen05) vs torch/cuBLAS per shape
"""
import ctypes as C
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2305_13484_b200 import _lib

lib = _lib.load()
lib.fl_gemm_set_rearm(0)   # one workspace for every call: the flags self-reset
ws = torch.empty(lib.fl_gemm_workspace_bytes(), dtype=torch.uint8, device="cuda")
REPS = 50
shapes = [(48, 2304, 768), (48, 768, 768), (48, 3072, 768), (48, 768, 3072), (48, 50257, 768),
          (112, 2304, 768), (112, 768, 3072), (1, 768, 3072), (100, 12288, 4096), (100, 4096, 16384)]
if len(sys.argv) > 1:
    shapes = [tuple(map(int, a.split("x"))) for a in sys.argv[1:]]
s = torch.cuda.Stream()
dbg = torch.zeros(4 * 8192, dtype=torch.int64, device="cuda")
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
        d = dbg.view(-1, 4).cpu().double()
        g = int((d[:2048, 1] > 0).sum().item() + (d[:2048, 3] > 0).sum().item() // 1)
        p = d[:2048][d[:2048, 1] > 0]
        lead = d[:2048, 3] > 0
        m = d[:2048][lead]
        te = d[2048:4096, 0][lead]
        e = d[4096:6144]
        ok = e[:, 1] > 0
        e = e[ok]
        ef = d[6144:8192, 0][ok]
        eb = d[6144:8192, 1][ok]
        ep = d[6144:8192, 2][ok]
        el = d[6144:8192, 3][ok]
        t0 = e[:, 0].min()
        print(f"   producer: {len(p)} CTAs, waits {100*p[:,0].sum()/max(p[:,1].sum(),1):.0f}% of {p[:,1].mean():.0f} clk;"
              f" mma: {len(m)} CTAs, full-waits {100*m[:,2].sum()/max(m[:,3].sum(),1):.0f}%, tmem-waits "
              f"{100*te.sum()/max(m[:,3].sum(),1):.0f}% of {m[:,3].mean():.0f} clk", flush=True)
        print(f"   epilogue: start spread {(e[:,0].max()-t0)/1e3:.1f} us, end {(e[:,1].min()-t0)/1e3:.1f}..{(e[:,1].max()-t0)/1e3:.1f} us;"
              f" tfull-wait {e[:,2].mean():.0f} clk, flag-wait {ef.mean():.0f} (max {ef.max():.0f}) clk, blocks {eb.mean():.0f} (ldtm {el.mean():.0f}, ldtm+sts {e[:,3].mean():.0f}) post {ep.mean():.0f}", flush=True)
