"""GEMM-only replay of one fused GPT-J decode step with cold weights.

    python tools/layer_gemm_bench.py [M ...]      (MODEL=gpt2: the C2 shapes)

28 layers x (QKV store, attn-out residual-add, FFN-up GELU, FFN-down
residual-add) + the LM head with the fused greedy argmax, each layer with its
own weights (11.3 GB: every weight byte comes from HBM, as in the real step),
captured in one CUDA graph; ours (C-ABI fl_gemm) vs torch.matmul (cuBLAS,
plain GEMMs without the epilogues).
"""
import ctypes as C
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2305_13484_b200 import _lib

lib = _lib.load()
lib.fl_gemm_set_rearm(0)   # one workspace for every call: the flags self-reset
for kv in filter(None, (os.environ.get("TUNE") or "").split(",")):   # diagnostics: fl_gemm_tune key=value
    k, v = kv.split("=")
    lib.fl_gemm_tune(int(k), int(v))
ws = torch.empty(lib.fl_gemm_workspace_bytes(), dtype=torch.uint8, device="cuda")
L, d, F, V = 28, 4096, 16384, 50400
if os.environ.get("MODEL") == "gpt2":     # C2 shapes (GPT-2 small)
    L, d, F, V = 12, 768, 3072, 50257
g = torch.Generator(device="cuda").manual_seed(0)
W = [[(torch.randn(n, k, device="cuda", generator=g) * 0.02).bfloat16() for n, k in
      ((3 * d, d), (d, d), (F, d), (d, F))] for _ in range(L)]
Wlm = (torch.randn(V, d, device="cuda", generator=g) * 0.02).bfloat16()
TILED = os.environ.get("TILED", "1") != "0"     # weights in the fl_tile_weight layout (as the executor runs)
WT = None
if TILED:
    def _tile(w):
        n, k = w.shape
        t = torch.empty(lib.fl_tiled_weight_bytes(n, k) // 2, dtype=torch.bfloat16, device="cuda")
        _lib.check(lib.fl_tile_weight(C.c_void_p(w.data_ptr()), n, k, C.c_void_p(t.data_ptr()), None))
        return t
    WT = [[_tile(w) for w in lw] for lw in W]
    torch.cuda.synchronize()
QF = "qf" in (os.environ.get("ONLY") or "")     # QKV and FFN-up as one GEMM over [W_qkv; W_fc]
if QF:
    WQF = [torch.cat([lw[0], lw[2]], 0) for lw in W]
    WQFT = [_tile(w) for w in WQF] if TILED else None
    torch.cuda.synchronize()
s = torch.cuda.Stream()
Ms = [int(a) for a in sys.argv[1:]] or [8, 64, 128, 192, 256, 320]
ONLY = os.environ.get("ONLY")      # e.g. "qkv" or "qkv,o": only these projections (28 cold layers)
SEL = ONLY.split(",") if ONLY else ["qkv", "o", "fc", "proj"]
for M in Ms:
    h = torch.randn(M, d, device="cuda").bfloat16()
    qkv = torch.empty(M, 3 * d, device="cuda", dtype=torch.bfloat16)
    f = torch.empty(M, F, device="cuda", dtype=torch.bfloat16)
    qf = torch.empty(M, 3 * d + F, device="cuda", dtype=torch.bfloat16)
    a = torch.randn(M, d, device="cuda").bfloat16()
    x = torch.zeros(M, d, device="cuda")
    keys = torch.zeros(M, device="cuda", dtype=torch.int64)
    st = C.c_void_p(0)
    def gemm(xx, ww, out, epi, ldo, wt=None):
        Mx, K = xx.shape
        N = ww.shape[0]
        wp = wt.data_ptr() if wt is not None else ww.data_ptr()
        _lib.check(lib.fl_gemm(xx.data_ptr(), K, wp, None, out.data_ptr(), ldo, Mx, N, K, epi, 1,
                               2 if wt is not None else 1,
                               ws.data_ptr(), C.c_void_p(torch.cuda.current_stream().cuda_stream)))
    def ours():
        for l in range(L):
            if "qkv" in SEL: gemm(h, W[l][0], qkv, 0, 3 * d, WT[l][0] if WT else None)
            if "o" in SEL: gemm(a, W[l][1], x, 2, d, WT[l][1] if WT else None)
            if "fc" in SEL: gemm(h, W[l][2], f, 1, F, WT[l][2] if WT else None)
            if "qf" in SEL: gemm(h, WQF[l], qf, 0, 3 * d + F, WQFT[l] if WQFT else None)
            if "proj" in SEL: gemm(f, W[l][3], x, 2, d, WT[l][3] if WT else None)
    def ref():
        for l in range(L):
            if "qkv" in SEL: torch.matmul(h, W[l][0].T, out=qkv)
            if "o" in SEL: torch.matmul(a, W[l][1].T)
            if "fc" in SEL: torch.matmul(h, W[l][2].T, out=f)
            if "qf" in SEL: torch.matmul(h, WQF[l].T, out=qf)
            if "proj" in SEL: torch.matmul(f, W[l][3].T)
    res = []
    for name, fn in (("ours", ours), ("cublas", ref)):
        with torch.cuda.stream(s):
            fn(); torch.cuda.synchronize()
            gr = torch.cuda.CUDAGraph()
            with torch.cuda.graph(gr, stream=s):
                fn()
            gr.replay(); torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(s)
            for _ in range(5):
                gr.replay()
            e1.record(s); torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / 5
        wel = sum({"qkv": 3 * d * d, "o": d * d, "fc": d * F, "proj": d * F, "qf": 3 * d * d + d * F}[k] for k in SEL)
        tf = 2 * M * L * wel / (ms * 1e-3) / 1e12
        gb = L * wel * 2 / (ms * 1e-3) / 1e9
        res.append(f"{name} {1e3 * ms / L:7.1f} us/layer ({tf:5.0f} TF/s, {gb:5.0f} GB/s weights)")
    print(f"{ONLY or 'all'} M={M:4d}  " + "   ".join(res), flush=True)
    if os.environ.get("GEMM_DBG"):
        dbg = torch.zeros(4 * 16384, dtype=torch.int64, device="cuda")
        lib.fl_gemm_debug(C.c_void_p(dbg.data_ptr())); ours(); torch.cuda.synchronize(); lib.fl_gemm_debug(None)
        dd = dbg.view(-1, 4).cpu().double()
        p = dd[:2048][dd[:2048, 1] > 0]
        lead = dd[:2048, 3] > 0
        m = dd[:2048][lead]
        lat = dd[2048:4096, 1][lead]
        e = dd[4096:6144]
        ok = e[:, 1] > 0
        e = e[ok]
        t0 = e[:, 0].min()
        print(f"   last GEMM: {len(p)} CTAs; producer waits {100*p[:,0].sum()/max(p[:,1].sum(),1):.0f}% of {p[:,1].mean():.0f} clk;"
              f" mma full-waits {100*m[:,2].sum()/max(m[:,3].sum(),1):.0f}% of {m[:,3].mean():.0f} clk; issue->full {lat.mean():.0f} clk;"
              f" CTA start spread {(e[:,0].max()-t0)/1e3:.1f} us, end {(e[:,1].min()-t0)/1e3:.1f}..{(e[:,1].max()-t0)/1e3:.1f} us;"
              f" tfull-wait {e[:,2].mean():.0f} clk, epi total {e[:,3].mean():.0f} clk", flush=True)
        t = dd[8192:8192 + 2048]
        ok2 = (t[:, 3] > 0) & (dd[4096:6144, 0] > 0)
        g0 = dd[4096:6144, 0][ok2]
        T0 = g0.min()
        tl = t[ok2]
        def rng(v):
            v = v[v > 0] - T0
            return f"{v.min()/1e3:.2f}..{v.max()/1e3:.2f}" if len(v) else "-"
        print(f"   timeline us (from first CTA start): start {rng(g0)} | X after pdl_wait {rng(tl[:,0])} |"
              f" last MMA {rng(tl[:,1])} | epi got acc {rng(tl[:,2])} | epi end {rng(dd[4096:6144,1][ok2])} |"
              f" dealloc {rng(tl[:,3])}", flush=True)
        raw = dbg.view(-1).cpu().double()
        for b in range(0, 4, 2):
            fulls = raw[4 * 10240 + b * 32: 4 * 10240 + b * 32 + 32]
            xs = raw[4 * 12288 + b * 32: 4 * 12288 + b * 32 + 32]
            ws_ = raw[4 * 14336 + b * 32: 4 * 14336 + b * 32 + 32]
            f = lambda v: " ".join(f"{(x - T0) / 1e3:.2f}" for x in v.tolist() if x > 0)
            print(f"   CTA {b}: W issue [{f(ws_)}]\n          X issue [{f(xs)}]\n          full    [{f(fulls)}]", flush=True)
        e6 = dd[6144:8192][ok2]
        print(f"   epi clk means: wait {e[:, 2].mean():.0f} flag {e6[:, 0].mean():.0f} blk {e6[:, 1].mean():.0f} post {e6[:, 2].mean():.0f} ld {e6[:, 3].mean():.0f}", flush=True)
        pro = raw[4 * 9216: 4 * 9216 + 4 * 148].view(-1, 4)[ok2[:148]]
        print(f"   prologue: ranges {rng(pro[:,0])} | alloc {rng(pro[:,1])} | init {rng(pro[:,2])} | cluster sync {rng(pro[:,3])}", flush=True)
