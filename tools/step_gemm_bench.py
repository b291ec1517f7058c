"""GEMM-only replay of the C3 (GPT-J 6B) fused step as the executor runs it.

    python tools/step_gemm_bench.py [M ...]        (env: MODEL=neox for C4 shapes)

Per layer: the merged in-projection (QKV + FFN-up over [W_qkv; W_fc], dual
operand, GELU on the FFN half) and the merged out-projection (attn-out +
FFN-down over K = Dl + Fl, residual add), each layer with its own tiled
weights (every weight byte from HBM, as in the real step), plus the LM head
with the fused argmax; captured in one CUDA graph.  Ours (fl_gemm2) vs
torch.matmul (cuBLAS) plain GEMMs of the same shapes.  Prints µs per layer,
the HBM fraction of the weight stream and the tensor fraction, against
MEASURED_PEAKS.json.
"""
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
# TUNE="0=0,3=1": fl_gemm_tune(key, value) pairs (0 = PDL, 1 max pairs, 2 stages, 3 kpb, 4 min units)
for kv in filter(None, (os.environ.get("TUNE") or "").split(",")):
    k, v = kv.split("=")
    lib.fl_gemm_tune(int(k), int(v))
peaks = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json"))) if os.path.exists(
    os.path.join(ROOT, "MEASURED_PEAKS.json")) else {"hbm_gbs": 6650.0, "bf16_tflops_sustained": 1400.0}
HBM, TF = peaks["hbm_gbs"], peaks.get("bf16_tflops_sustained", 1400.0)
ws = torch.empty(lib.fl_gemm_workspace_bytes(), dtype=torch.uint8, device="cuda")
if os.environ.get("MODEL", "gptj") == "neox":
    L, d, F, V = 44, 6144, 24576, 50432
else:
    L, d, F, V = 28, 4096, 16384, 50400
q3 = 3 * d
g = torch.Generator(device="cuda").manual_seed(0)


def tile(w):
    n, k = w.shape
    t = torch.empty(lib.fl_tiled_weight_bytes(n, k) // 2, dtype=torch.bfloat16, device="cuda")
    _lib.check(lib.fl_tile_weight(C.c_void_p(w.data_ptr()), n, k, C.c_void_p(t.data_ptr()), None))
    return t


Win = [(torch.randn(q3 + F, d, device="cuda", generator=g) * 0.02).bfloat16() for _ in range(L)]
Wout = [(torch.randn(d, d + F, device="cuda", generator=g) * 0.02).bfloat16() for _ in range(L)]
Wlm = (torch.randn(V, d, device="cuda", generator=g) * 0.02).bfloat16()
WinT = [tile(w) for w in Win]
WoutT = [tile(w) for w in Wout]
WlmT = tile(Wlm)
torch.cuda.synchronize()
s = torch.cuda.Stream()
Ms = [int(a) for a in sys.argv[1:]] or [8, 32, 64, 96, 128, 160, 192, 256, 320]
SEL = (os.environ.get("ONLY") or "in,out,lm").split(",")
for M in Ms:
    h = torch.randn(M, d, device="cuda").bfloat16()
    h2 = torch.randn(M, d, device="cuda").bfloat16()
    act = torch.randn(M, 4 * d + F, device="cuda").bfloat16()      # [q|k|v | a | f]
    x = torch.zeros(M, d, device="cuda")
    keys = torch.zeros(M, device="cuda", dtype=torch.int64)

    def g2(xx, x2, w, out, ldo, N, K, epi, ldx, nsplit=0, ogap=0, kp=None):
        _lib.check(lib.fl_gemm2(xx.data_ptr(), x2.data_ptr() if x2 is not None else None, ldx, w.data_ptr(), None,
                                out.data_ptr() if out is not None else None, ldo, M, N, K, epi, 1, 2, nsplit, ogap,
                                kp.data_ptr() if kp is not None else None, 0, ws.data_ptr(),
                                C.c_void_p(torch.cuda.current_stream().cuda_stream)))

    def ours():
        for l in range(L):
            if "in" in SEL:
                g2(h, h2, WinT[l], act, 4 * d + F, q3 + F, d, 1, d, nsplit=q3, ogap=d)
            if "out" in SEL:
                g2(act[:, q3:], None, WoutT[l], x, d, d, d + F, 2, 4 * d + F)
        if "lm" in SEL:
            g2(h, None, WlmT, None, 0, V, d, 4, d, kp=keys)

    def ref():
        for l in range(L):
            if "in" in SEL:
                torch.matmul(h, Win[l].T)
            if "out" in SEL:
                torch.matmul(act[:, q3:], Wout[l].T)
        if "lm" in SEL:
            torch.matmul(h, Wlm.T)

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
        ms = e0.elapsed_time(e1) / 5
        wel = L * ((q3 + F) * d * ("in" in SEL) + d * (d + F) * ("out" in SEL)) + V * d * ("lm" in SEL)
        gb = wel * 2 / (ms * 1e-3) / 1e9
        tf = 2 * M * wel / (ms * 1e-3) / 1e12
        res.append(f"{name} {1e3 * ms:8.1f} us ({gb:5.0f} GB/s = {gb / HBM:4.2f} HBM, {tf:5.0f} TF/s = {tf / TF:4.2f})")
    print(f"{','.join(SEL)} M={M:4d}  " + "   ".join(res), flush=True)
    if os.environ.get("GEMM_DBG"):
        # in-kernel clocks of the LAST GEMM of ours(): per CTA producer wait /
        # total, MMA full-barrier wait / total, mean weight issue -> full
        dbg2 = torch.zeros(2 * 4 * 16384, dtype=torch.int64, device="cuda")
        dbg = dbg2[:4 * 16384]
        lib.fl_gemm_tune(9, 1)    # alternate halves: the last two launches
        lib.fl_gemm_debug(C.c_void_p(dbg.data_ptr()))
        ours()
        torch.cuda.synchronize()
        lib.fl_gemm_debug(None)
        dd = dbg.view(-1, 4).cpu().double()
        p = dd[:2048][dd[:2048, 1] > 0]
        lead = dd[:2048, 3] > 0
        m = dd[:2048][lead]
        lat = dd[2048:4096, 1][lead]
        tw = dd[2048:4096, 0][lead]
        e = dd[4096:6144]
        e = e[e[:, 1] > 0]
        t0 = e[:, 0].min()
        print(f"   last GEMM: {len(p)} producer CTAs; producer waits {100 * p[:, 0].sum() / max(p[:, 1].sum(), 1):.0f}%"
              f" of {p[:, 1].mean():.0f} clk; mma full-waits {100 * m[:, 2].sum() / max(m[:, 3].sum(), 1):.0f}%"
              f" of {m[:, 3].mean():.0f} clk (tmem-empty waits {tw.mean():.0f}); issue->full {lat.mean():.0f} clk;"
              f" CTA start spread {(e[:, 0].max() - t0) / 1e3:.1f} us, end {(e[:, 1].min() - t0) / 1e3:.1f}.."
              f"{(e[:, 1].max() - t0) / 1e3:.1f} us; epi tfull-wait {e[:, 2].mean():.0f} clk, epi total {e[:, 3].mean():.0f}",
              flush=True)
        ok2 = (dd[8192:8192 + 2048, 3] > 0) & (dd[4096:6144, 0] > 0)
        g0 = dd[4096:6144, 0][ok2]
        T0 = g0.min()
        tl = dd[8192:8192 + 2048][ok2]

        def rng(v):
            v = v[v > 0] - T0
            return f"{v.min() / 1e3:.2f}..{v.max() / 1e3:.2f}" if len(v) else "-"
        raw = dbg.view(-1).cpu().double()
        pro = raw[4 * 9216: 4 * 9216 + 4 * 148].view(-1, 4)[ok2[:148]]
        print(f"   timeline us: start {rng(g0)} | prologue done {rng(pro[:, 3])} | X after pdl_wait {rng(tl[:, 0])} |"
              f" last MMA {rng(tl[:, 1])} | epi got acc {rng(tl[:, 2])} | epi end {rng(dd[4096:6144, 1][ok2])} |"
              f" dealloc {rng(tl[:, 3])}", flush=True)
        ends = (dd[4096:6144, 1][ok2] - T0) / 1e3
        print("   epi end quantiles us: " + " ".join(f"{q:.2f}" for q in torch.quantile(ends, torch.tensor([0.0, 0.1, 0.5, 0.9, 1.0], dtype=ends.dtype)).tolist()), flush=True)
        # the last two launches (alternating halves): predecessor end -> successor start
        halves = [dbg2[i * 4 * 16384:(i + 1) * 4 * 16384].view(-1, 4).cpu().double() for i in range(2)]
        info = []
        for hv in halves:
            ok = (hv[4096:6144, 0] > 0) & (hv[8192:8192 + 2048, 3] > 0)
            if ok.any():
                info.append((hv[4096:6144, 0][ok].min(), hv[4096:6144, 0][ok].max(), hv[8192:8192 + 2048, 0][ok].max(),
                             hv[4096:6144, 1][ok].max(), hv[8192:8192 + 2048, 3][ok].max(), int(ok.sum())))
        if len(info) == 2:
            info.sort()
            a_, b_ = info
            Z = a_[0]
            f = lambda t: f"{(t - Z) / 1e3:.2f}"
            print(f"   pair of launches (us from the first's first CTA): first [{a_[5]} CTAs] start {f(a_[0])}..{f(a_[1])},"
                  f" X ready {f(a_[2])}, epi end {f(a_[3])}, last dealloc {f(a_[4])} | second [{b_[5]} CTAs] start"
                  f" {f(b_[0])}..{f(b_[1])}, X ready {f(b_[2])}, epi end {f(b_[3])}, last dealloc {f(b_[4])}", flush=True)
