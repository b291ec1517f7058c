"""A stand-in for the CUDA library and torch.cuda so the REAL executor host
path (CudaExecutor: row tables, prompt rows, shuffles, imports, the device
clock and its TP agreement) runs on CPU.  Test infrastructure only: nothing
is computed -- every fl_* call is recorded and returns FL_OK; events report a
deterministic, rank-dependent 'device' time.

    with stub_device(rank=0) as rec:
        ex = CudaExecutor(spec, prompts, device="cpu", ...)
        ...
    rec.steps  -> [(n_rows, n_dec, rows_changed, sha of the row table)]
"""

from __future__ import annotations

import contextlib
import ctypes as C
import hashlib

import numpy as np


class _Rec:
    def __init__(self, rank):
        self.rank = rank
        self.calls = []
        self.steps = []
        self.shuffles = []
        self.comm = None
        self.n_events = 0


class StubLib:
    def __init__(self, rec: _Rec):
        self._rec = rec

    def __getattr__(self, name):
        if not name.startswith("fl_"):
            raise AttributeError(name)
        rec = self._rec

        def call(*a):
            rec.calls.append(name)
            if name == "fl_workspace_bytes":
                return 4096
            if name == "fl_tiled_weight_bytes":
                n, k = a
                return (n + 127) // 128 * 128 * k * 2
            if name == "fl_create":
                a[2]._obj.value = 0x1000 + rec.rank
            elif name == "fl_comm_init":
                rec.comm = (bytes(a[1].raw[:128]), a[2], a[3])
            elif name == "fl_step":
                _, rows, n, n_dec, changed = a[:5]
                flat = np.ctypeslib.as_array(C.cast(rows, C.POINTER(C.c_int32)), shape=(n * 6,)).copy()
                rec.steps.append((n, n_dec, changed, hashlib.sha256(flat.tobytes()).hexdigest()[:16]))
            elif name == "fl_shuffle":
                _, moves, n = a[:3]
                rec.shuffles.append(tuple(moves[i] for i in range(3 * n)))
            elif name == "fl_kernel_launches":
                return len(rec.steps)
            elif name == "fl_abi_version":
                return 1
            elif name == "fl_last_error":
                return b"stub"
            return 0
        return call


class _Stream:
    cuda_stream = 0

    def __init__(self, *a, **k):
        pass

    def synchronize(self):
        pass

    def wait_event(self, ev):
        pass


class _Event:
    def __init__(self, rec, enable_timing=False):
        self._rec = rec
        rec.n_events += 1
        self._k = rec.n_events

    def record(self, stream=None):
        pass

    def synchronize(self):
        pass

    def query(self):
        return True

    def elapsed_time(self, end):
        # a rank-dependent 'device' time: the ranks' schedules must still agree
        return 1.0 + 0.25 * self._rec.rank + 0.01 * (end._k % 7)


class StubCuda:
    def __init__(self, rec: _Rec):
        self._rec = rec
        self.Stream = _Stream

    def Event(self, enable_timing=False):
        return _Event(self._rec, enable_timing)

    def synchronize(self, *a):
        pass

    def current_stream(self, *a):
        return _Stream()

    def mem_get_info(self, *a):
        return (8 << 30, 16 << 30)

    @contextlib.contextmanager
    def stream(self, s):
        yield


@contextlib.contextmanager
def stub_device(rank: int = 0):
    from paper_2305_13484_b200 import _lib
    from paper_2305_13484_b200 import executor as exmod
    rec = _Rec(rank)
    saved = (_lib.load, exmod._cuda)
    lib = StubLib(rec)
    _lib.load = lambda: lib
    exmod._cuda = StubCuda(rec)
    try:
        yield rec
    finally:
        _lib.load, exmod._cuda = saved
