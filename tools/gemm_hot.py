"""L2-resident GEMM rate: one [N, K] weight (fits L2) multiplied again and again,
so HBM is out of the picture and the pipeline (TMA issue, smem, MMA) is what
is timed.  python tools/gemm_hot.py [M ...]  (env N, K, TUNE as step_gemm_bench)"""
import ctypes as C
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2305_13484_b200 import _lib  # noqa: E402

lib = _lib.load()
lib.fl_gemm_set_rearm(0)
for kv in filter(None, (os.environ.get("TUNE") or "").split(",")):
    k, v = kv.split("=")
    lib.fl_gemm_tune(int(k), int(v))
N, K = int(os.environ.get("N", 8192)), int(os.environ.get("K", 4096))
ws = torch.empty(lib.fl_gemm_workspace_bytes(), dtype=torch.uint8, device="cuda")
w = (torch.randn(N, K, device="cuda") * 0.02).bfloat16()
wt = torch.empty(lib.fl_tiled_weight_bytes(N, K) // 2, dtype=torch.bfloat16, device="cuda")
_lib.check(lib.fl_tile_weight(C.c_void_p(w.data_ptr()), N, K, C.c_void_p(wt.data_ptr()), None))
s = torch.cuda.Stream()
for M in [int(a) for a in sys.argv[1:]] or [64, 128, 256, 320]:
    x = torch.randn(M, K, device="cuda").bfloat16()
    out = torch.empty(M, N, device="cuda").bfloat16()

    def ours():
        for _ in range(20):
            _lib.check(lib.fl_gemm2(x.data_ptr(), None, K, wt.data_ptr(), None, out.data_ptr(), N, M, N, K, 0, 1, 2,
                                    0, 0, None, 0, ws.data_ptr(), C.c_void_p(torch.cuda.current_stream().cuda_stream)))

    def ref():
        for _ in range(20):
            torch.matmul(x, w.T, out=out)
    res = []
    for name, fn in (("ours", ours), ("cublas", ref)):
        with torch.cuda.stream(s):
            fn()
            torch.cuda.synchronize()
            gr = torch.cuda.CUDAGraph()
            with torch.cuda.graph(gr, stream=s):
                fn()
            gr.replay()
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(s)
            for _ in range(5):
                gr.replay()
            e1.record(s)
            torch.cuda.synchronize()
        us = e0.elapsed_time(e1) / 100 * 1e3
        res.append(f"{name} {us:7.1f} us {2 * M * N * K / us / 1e6:6.0f} TF/s")
    print(f"hot N={N} K={K} M={M:4d}  " + "   ".join(res), flush=True)
    if os.environ.get("GEMM_DBG"):
        dbg = torch.zeros(4 * 8192, dtype=torch.int64, device="cuda")
        lib.fl_gemm_debug(C.c_void_p(dbg.data_ptr()))
        ours()
        torch.cuda.synchronize()
        lib.fl_gemm_debug(None)
        dd = dbg.view(-1, 4).cpu().double()
        p = dd[:2048][dd[:2048, 1] > 0]
        lead = dd[:2048, 3] > 0
        m = dd[:2048][lead]
        lat = dd[2048:4096, 1][lead]
        e = dd[4096:6144]
        ok = e[:, 1] > 0
        e, f = e[ok], dd[6144:8192][ok]
        t0 = e[:, 0].min()
        print(f"   {len(p)} CTAs: producer waits {100 * p[:, 0].sum() / max(p[:, 1].sum(), 1):.0f}% of {p[:, 1].mean():.0f} clk;"
              f" mma full-waits {100 * m[:, 2].sum() / max(m[:, 3].sum(), 1):.0f}% of {m[:, 3].mean():.0f} clk;"
              f" issue->full {lat.mean():.0f} clk; start spread {(e[:, 0].max() - t0) / 1e3:.1f} us,"
              f" end {(e[:, 1].min() - t0) / 1e3:.1f}..{(e[:, 1].max() - t0) / 1e3:.1f} us;"
              f" epi: tfull-wait {e[:, 2].mean():.0f}, total {e[:, 3].mean():.0f}, flag-wait {f[:, 0].mean():.0f},"
              f" blocks {f[:, 1].mean():.0f}, post {f[:, 2].mean():.0f}, tmem-ld {f[:, 3].mean():.0f} clk", flush=True)
