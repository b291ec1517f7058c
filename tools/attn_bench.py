"""K4 decode attention alone: bandwidth at steady-state-like contexts.

    python tools/attn_bench.py [rows] [hd] [heads] [maxctx]
"""
import ctypes as C
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2305_13484_b200 import _lib

M = int(sys.argv[1]) if len(sys.argv) > 1 else 340
hd = int(sys.argv[2]) if len(sys.argv) > 2 else 256
H = int(sys.argv[3]) if len(sys.argv) > 3 else 16
S = int(sys.argv[4]) if len(sys.argv) > 4 else 1055
lib = _lib.load()
g = torch.Generator(device="cuda").manual_seed(0)
kv = torch.randn((M, 2, H, S, hd), device="cuda", generator=g).bfloat16()
q = torch.randn((M, H * hd), device="cuda", generator=g).bfloat16()
ctx = torch.randint(32, S + 1, (M,), device="cuda", generator=g, dtype=torch.int32)
if os.environ.get("ORDER"):      # rows by descending context, as the step's row_order ranks them
    ctx = ctx.sort(descending=True).values.contiguous()
rows = torch.zeros((M, 6), dtype=torch.int32, device="cuda")
rows[:, 0] = torch.arange(M, dtype=torch.int32)
out = torch.empty_like(q)
ws = torch.empty(lib.fl_attention_workspace_bytes(M, H, hd, S), dtype=torch.uint8, device="cuda")
s = torch.cuda.current_stream()
def run():
    _lib.check(lib.fl_attention(q.data_ptr(), rows.data_ptr(), ctx.data_ptr(), M, H, hd, kv.data_ptr(), M, S,
                                out.data_ptr(), ws.data_ptr(), 1, C.c_void_p(s.cuda_stream)))
run(); torch.cuda.synchronize()
# reference on a few rows
ref_err = 0.0
for r in range(0, M, max(1, M // 8)):
    n = int(ctx[r])
    K = kv[r, 0, :, :n].float(); V = kv[r, 1, :, :n].float()
    qq = q[r].float().view(H, hd)
    p = torch.softmax((qq.unsqueeze(1) @ K.transpose(1, 2)).squeeze(1) / hd ** 0.5, dim=-1)
    o = (p.unsqueeze(1) @ V).squeeze(1).reshape(-1)
    ref_err = max(ref_err, (o - out[r].float()).abs().max().item())
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
R = 20
e0.record()
for _ in range(R):
    run()
e1.record(); torch.cuda.synchronize()
us = e0.elapsed_time(e1) * 1e3 / R
byt = int(ctx.sum()) * 2 * H * hd * 2 + M * 2 * H * hd * 2
print(f"attention M={M} hd={hd} H={H}: {us:.1f} us, {byt/1e6:.1f} MB, {byt/us/1e3:.0f} GB/s, max err {ref_err:.3e}")
if os.environ.get("ATT_DBG"):
    # per-CTA %globaltimer stamps of one launch (fl_attention_debug)
    nb = 2 * 148
    dbg = torch.zeros(64 * nb, dtype=torch.int64, device="cuda")
    lib.fl_attention_debug(C.c_void_p(dbg.data_ptr()))
    run()
    torch.cuda.synchronize()
    lib.fl_attention_debug(None)
    d = dbg.view(nb, 64).cpu().double()
    d = d[d[:, 0] > 0]
    T0 = d[:, 0].min()
    starts, pdl = (d[:, 0] - T0) / 1e3, (d[:, 1] - T0) / 1e3
    items, gaps, firsts, ends, counts = [], [], [], [], []
    for row in d:
        st = [(row[2 + 2 * i] - T0) / 1e3 for i in range(31) if row[3 + 2 * i] > 0]
        en = [(row[3 + 2 * i] - T0) / 1e3 for i in range(31) if row[3 + 2 * i] > 0]
        counts.append(len(st))
        if st:
            firsts.append(st[0])
            ends.append(en[-1])
        items += [e - s for s, e in zip(st, en)]
        gaps += [st[i + 1] - en[i] for i in range(len(st) - 1)]
    q = lambda v: "min %.2f med %.2f max %.2f" % (min(v), sorted(v)[len(v) // 2], max(v)) if v else "-"
    print(f"   CTAs {len(d)}: start {q(starts.tolist())} | dep wait done {q(pdl.tolist())} | first item {q(firsts)} |"
          f" end {q(ends)}")
    print(f"   items/CTA {q(counts)} | item us {q(items)} (mean {sum(items) / max(len(items), 1):.2f}) |"
          f" gap between items {q(gaps)} (mean {sum(gaps) / max(len(gaps), 1):.2f})", flush=True)
