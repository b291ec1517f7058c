"""K10 shuffle bandwidth probe: GPT-J-shape KV pool, n moves of ctx tokens.

    python tools/shuffle_bench.py [ctx] [moves]
"""
import ctypes as C
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2305_13484_b200 import _lib

ctx = int(sys.argv[1]) if len(sys.argv) > 1 else 512
nm = int(sys.argv[2]) if len(sys.argv) > 2 else 2
L, H, hd, S, Cs = 28, 16, 256, 1055, 16
lib = _lib.load()
kv = torch.zeros((L, Cs, 2, H, S, hd), dtype=torch.bfloat16, device="cuda")
dummy = kv.data_ptr()
layers = (C.c_void_p * (L * 12))(*([dummy] * (L * 12)))
m = _lib.ModelDesc(1, 1, L, 4096, H, hd, 16384, 50400, 2048, 64, 1e-5, 0, 1, dummy, None, dummy, dummy,
                   dummy, None, C.cast(layers, C.POINTER(C.c_void_p)))
st = torch.zeros(64, dtype=torch.int32, device="cuda")
p = _lib.PoolDesc(Cs, S, 64, 16, 8, 0, kv.data_ptr(), st.data_ptr(), st.data_ptr(), st.data_ptr(),
                  st.data_ptr(), None, 0)
nb = lib.fl_workspace_bytes(C.byref(m), C.byref(p))
ws = torch.empty(nb, dtype=torch.uint8, device="cuda")
p.workspace, p.workspace_bytes = ws.data_ptr(), nb
h = C.c_void_p()
_lib.check(lib.fl_create(C.byref(m), C.byref(p), C.byref(h)))
moves = []
for i in range(nm):
    moves += [2 * i + 1, 2 * i, ctx]
arr = (C.c_int32 * len(moves))(*moves)
s = torch.cuda.current_stream()
for _ in range(3):
    _lib.check(lib.fl_shuffle(h, arr, nm, C.c_void_p(s.cuda_stream)))
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
R = 20
e0.record()
for _ in range(R):
    _lib.check(lib.fl_shuffle(h, arr, nm, C.c_void_p(s.cuda_stream)))
e1.record(); torch.cuda.synchronize()
us = e0.elapsed_time(e1) * 1e3 / R
byt = 2 * nm * ctx * 2 * L * H * hd * 2
print(f"shuffle ctx={ctx} moves={nm}: {us:.1f} us, {byt/1e6:.1f} MB read+write, {byt/us/1e3:.0f} GB/s")
