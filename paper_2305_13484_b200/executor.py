"""CudaExecutor: runs the fused stream's iterations on the B200 via the C-ABI.

Plugged into ``FusionStream(..., executor=CudaExecutor(...))``, it realises
each modelled action of the reference loop on the device:

* ``try_fuse_pending`` (engine.py:97-124) -> ``on_fuse``: the request's prompt
  is queued as PREFILL rows of the next fused iteration (positions
  0..P-2) and its first DECODE row carries prompt token P-1 explicitly.
* ``step_iteration`` (engine.py:128-160) -> ``run_iteration``: one
  ``fl_step`` over the live window [buffer_offset, +buffer_size) in window
  order (orphaned slots of fusion_noshuffle become ORPHAN rows that are
  computed over stale KV and discarded -- the paper's naive scheme,
  PAPER.md:254) followed by the prefill rows.
* ``apply_shuffle`` (buffer.py:261-278) -> ``on_shuffle``: the plan's moves
  become (src, dst, live-length) triples for the K10 kernel.

Device memory is owned here through PyTorch: weights, the KV pool
[L][C][2][H/tp][S][hd], per-request state (next token / position / count /
token history, indexed rid % R) and the library workspace.  Logical slot s
lives in physical slot s % C; the live window never spans more than C slots
(checked every iteration, ``CapacityExceeded`` otherwise).

Because stop lengths are pre-sampled, the host never needs a generated token
to schedule: steady-state iterations upload nothing and read nothing back.
"""

from __future__ import annotations

import ctypes as C

import numpy as np
import torch

from . import _lib
from .errors import CapacityExceeded, InvalidParam
from .models import LAYER_KEYS, ModelSpec, init_weights

GEMM_KEYS = ("w_qkv", "w_o", "w_fc", "w_proj")

_TORCH_DTYPE = {"f32": torch.float32, "bf16": torch.bfloat16}
_PAD = (0, -1, -1, -1, _lib.ROW_ORPHAN, 1)
_ROW_P = C.POINTER(_lib.Row)
# streams / events / synchronisation go through this name, so the host path
# can be driven on CPU against a stub library (tests/test_tp_host.py)
_cuda = torch.cuda


def _pad_rows(a):
    """Pad an int32 [n, 6] row table to its bucket with PAD rows."""
    n = len(a)
    b = bucket(n)
    if b == n:
        return np.ascontiguousarray(a)
    out = np.empty((b, 6), dtype=np.int32)
    out[:n] = a
    out[n:] = _PAD
    return out


def _rows_ptr(a):
    return a.ctypes.data_as(_ROW_P)


def bucket(n: int) -> int:
    """Row-count buckets: each (rows, window) bucket pair is one CUDA graph;
    the padding rows are ORPHAN rows over one stale position (discarded)."""
    if n <= 0:
        return 0
    # padding rows cost GEMM time roughly in proportion (the weight stream
    # is shared, but MMA and epilogue work grow with the window): 16-row
    # steps up to 256 rows, 32 beyond
    for limit, step in ((64, 8), (256, 16)):
        if n <= limit:
            return -(-n // step) * step
    return -(-n // 32) * 32


class CudaExecutor:
    def __init__(self, spec: ModelSpec, prompts, *, dtype: str = "bf16", pool_slots: int = 128,
                 max_rows: int | None = None, max_seq: int | None = None,
                 max_new_tokens: int = 1024, input_len: int | None = None,
                 state_slots: int = 4096, tp_rank: int = 0, tp_size: int = 1, seed: int = 0,
                 weights: dict | None = None, use_tensor_cores: bool | None = None,
                 capture_logits: bool = False, device: str = "cuda", comm_id: bytes | None = None,
                 time_steps: bool = False, use_graphs: bool = True, device_plan: bool = False,
                 tiled: bool | None = None, merged_in: bool | None = None,
                 merged_out: bool | None = None, merged_in_max_rows: int = -1,
                 prefill: str = "inline", prefill_slots: int = 32, eos_token: int | None = None):
        if dtype not in _TORCH_DTYPE:
            raise InvalidParam(f"dtype must be f32 or bf16, got {dtype}")
        if prefill not in ("inline", "side"):
            raise InvalidParam(f"prefill must be 'inline' or 'side', got {prefill!r}")
        self.lib = _lib.load()
        # data-dependent stop: a request finishes when its greedy
        # token equals eos_token (or at max_output_length); None = the
        # reference's pre-sampled actual_output_length
        self.eos_token = None if eos_token is None else int(eos_token)
        self._tok_host = None
        # plan AND execute every shuffle boundary on the device (fl_shuffle_planned)
        self.device_plan = bool(device_plan)
        self._plan_host = None
        self.device_plans = 0
        self.spec = spec
        self.prompts = prompts
        self.dtype = dtype
        self.tp_rank, self.tp_size = tp_rank, tp_size
        self.device = torch.device(device)
        self._auto_pool = not pool_slots
        self.C = pool_slots or 1
        self.R = state_slots
        self.max_new = max_new_tokens
        if max_seq is None:
            if input_len is None:
                raise InvalidParam("need max_seq or input_len")
            max_seq = input_len + max_new_tokens - 1
        self.S = max_seq
        if spec.family == "gpt2" and max_seq > spec.max_pos:
            # learned positions: a row at pos >= max_pos would read past wpe
            raise InvalidParam(f"max_seq {max_seq} > {spec.name} max_pos {spec.max_pos}")
        self.max_rows = bucket(max_rows or (pool_slots + 16 * (input_len or 32)))
        if self.max_rows < bucket(pool_slots) + 64:
            self.max_rows = bucket(bucket(pool_slots) + 64)
        if use_tensor_cores is None:
            use_tensor_cores = dtype == "bf16"
        self.use_tc = bool(use_tensor_cores)
        tdt = _TORCH_DTYPE[dtype]
        hl = spec.n_head // tp_size

        # ---- weights (this rank's shard)
        if weights is None:
            weights = init_weights(spec, seed=seed, device=self.device, dtype=tdt, rank=tp_rank,
                                   world=tp_size)
        self.w = {k: v.to(self.device, tdt).contiguous() for k, v in weights.items()}
        # tensor-core path: projection weights in the GEMM's tiled layout
        # (fl_tile_weight: every 128 x 64 tile the GEMM streams is contiguous);
        # the caller's tensors are left untouched, our own copies are replaced
        self.tiled = self.use_tc if tiled is None else bool(tiled) and self.use_tc
        parallel = spec.family in ("gptj", "neox")
        # parallel residual (gptj, neox): attn-out and FFN-down as one GEMM over
        # K = Dl + Fl with W_cat = [W_o | W_proj] and b_o + b_proj, i.e. ONE
        # all-reduce per layer under TP.  Default: on at tp 1; under TP the
        # north star's layout (an all-reduce after attn-out AND after FFN-down)
        if merged_out is None:
            merged_out = tp_size == 1
        self.merged = bool(merged_out) and self.use_tc and parallel
        self.tp_layout = ("one all-reduce per layer (merged attn-out + FFN-down)" if self.merged
                          else "two all-reduces per layer (after attn-out and after FFN-down)")
        self._wcat, self._bcat = [], []
        # ... and QKV and FFN-up as one GEMM over [W_qkv; W_fc] (rows 3*Dl..
        # read the MLP input, get GELU, land after the attention output)
        if merged_in is None:
            merged_in = True
        self.merged_in = (bool(merged_in) and self.use_tc and parallel
                          and (3 * hl * spec.head_dim) % 256 == 0)
        self.merged_in_max_rows = merged_in_max_rows
        self._win, self._bin = [], []
        if self.merged_in:
            for l in range(spec.n_layer):
                wq, wf = self.w.pop(f"layers.{l}.w_qkv"), self.w.pop(f"layers.{l}.w_fc")
                self.w[f"layers.{l}.w_in"] = torch.cat([wq, wf], dim=0).contiguous()
                bq, bf = self.w.pop(f"layers.{l}.b_qkv", None), self.w.pop(f"layers.{l}.b_fc", None)
                if bq is not None or bf is not None:
                    bq = bq if bq is not None else torch.zeros(wq.shape[0], dtype=tdt, device=self.device)
                    bf = bf if bf is not None else torch.zeros(wf.shape[0], dtype=tdt, device=self.device)
                    self.w[f"layers.{l}.b_in"] = torch.cat([bq, bf]).contiguous()
                del wq, wf, bq, bf
        if self.merged:
            for l in range(spec.n_layer):
                wo, wp = self.w.pop(f"layers.{l}.w_o"), self.w.pop(f"layers.{l}.w_proj")
                self.w[f"layers.{l}.w_cat"] = torch.cat([wo, wp], dim=1).contiguous()
                del wo, wp
                bs = [b.float() for b in (self.w.get(f"layers.{l}.b_o"), self.w.get(f"layers.{l}.b_proj"))
                      if b is not None]
                if bs:
                    self.w[f"layers.{l}.b_cat"] = sum(bs).to(tdt)
        if self.tiled:
            names = [f"layers.{l}.{k}" for l in range(spec.n_layer) for k in GEMM_KEYS + ("w_cat", "w_in")] + ["w_lm"]
            for name in names:
                t = self.w.get(name)
                if t is None:
                    continue
                n, k = t.shape
                tt = torch.empty(self.lib.fl_tiled_weight_bytes(n, k) // 2, dtype=tdt, device=self.device)
                _lib.check(self.lib.fl_tile_weight(C.c_void_p(t.data_ptr()), n, k, C.c_void_p(tt.data_ptr()),
                                                   C.c_void_p(_cuda.current_stream(self.device).cuda_stream)))
                self.w[name] = tt
                del t
        if self.merged_in:
            # windows wider than the library's merged_in_max_rows run QKV and
            # FFN-up apart over views of the stacked weight (rows 3*Dl.. start
            # at element 3*Dl*d in both the row-major and the tiled layout)
            q3 = 3 * hl * spec.head_dim
            for l in range(spec.n_layer):
                wi = self.w[f"layers.{l}.w_in"].view(-1)
                self.w[f"layers.{l}.w_qkv"] = wi[:q3 * spec.d_model]
                self.w[f"layers.{l}.w_fc"] = wi[q3 * spec.d_model:]
                bi = self.w.get(f"layers.{l}.b_in")
                if bi is not None:
                    self.w[f"layers.{l}.b_qkv"], self.w[f"layers.{l}.b_fc"] = bi[:q3], bi[q3:]
        del weights       # our own row-major copies are freed before the KV pool is sized
        ptrs = []
        for layer in range(spec.n_layer):
            for key in LAYER_KEYS:
                t = self.w.get(f"layers.{layer}.{key}")
                ptrs.append(t.data_ptr() if t is not None else None)
        self._layer_ptrs = (C.c_void_p * len(ptrs))(*ptrs)

        def ptr(name):
            t = self.w.get(name)
            return t.data_ptr() if t is not None else None

        self.mdesc = _lib.ModelDesc(
            _lib.FL_FAMILY[spec.family], _lib.FL_DTYPE[dtype], spec.n_layer, spec.d_model,
            spec.n_head, spec.head_dim, spec.d_ff, spec.vocab, spec.max_pos, spec.rotary_dim,
            spec.ln_eps, tp_rank, tp_size, ptr("wte"), ptr("wpe"), ptr("lnf_g"), ptr("lnf_b"),
            ptr("w_lm"), ptr("b_lm"), C.cast(self._layer_ptrs, C.POINTER(C.c_void_p)))

        # ---- KV pool and per-request state
        if self._auto_pool:
            # as many slots as fit in free HBM after weights, keeping 6 GB for
            # the workspace and the allocator
            es = 2 if dtype == "bf16" else 4
            slot = spec.n_layer * 2 * hl * self.S * spec.head_dim * es
            free, _ = _cuda.mem_get_info(self.device)
            self.C = max(1, min(state_slots, int((free - 6 * 2**30) // slot)))
            self.max_rows = bucket(max_rows or (self.C + 16 * (input_len or 32)))
            if self.max_rows < bucket(self.C) + 64:
                self.max_rows = bucket(bucket(self.C) + 64)
        self.kv = torch.empty((spec.n_layer, self.C, 2, hl, self.S, spec.head_dim), dtype=tdt,
                              device=self.device)
        i32 = dict(dtype=torch.int32, device=self.device)
        self.req_tok = torch.zeros(self.R, **i32)
        self.req_pos = torch.zeros(self.R, **i32)
        self.req_ngen = torch.zeros(self.R, **i32)
        self.tok_hist = torch.zeros((self.R, self.max_new), **i32)
        self.pdesc = _lib.PoolDesc(self.C, self.S, self.max_rows, self.R, self.max_new,
                                   (2 if self.tiled else 1) if self.use_tc else 0, self.kv.data_ptr(),
                                   self.req_tok.data_ptr(),
                                   self.req_pos.data_ptr(), self.req_ngen.data_ptr(),
                                   self.tok_hist.data_ptr(), None, 0)
        nbytes = self.lib.fl_workspace_bytes(C.byref(self.mdesc), C.byref(self.pdesc))
        if nbytes == 0:
            _lib.check(-1)
        self.ws = torch.empty(nbytes, dtype=torch.uint8, device=self.device)
        self.pdesc.workspace = self.ws.data_ptr()
        self.pdesc.workspace_bytes = nbytes
        h = C.c_void_p()
        _lib.check(self.lib.fl_create(C.byref(self.mdesc), C.byref(self.pdesc), C.byref(h)))
        self.handle = h
        if self.merged:
            wc = [self.w[f"layers.{l}.w_cat"].data_ptr() for l in range(spec.n_layer)]
            bc = [self.w[f"layers.{l}.b_cat"].data_ptr() if f"layers.{l}.b_cat" in self.w else None
                  for l in range(spec.n_layer)]
            self._wcat = (C.c_void_p * len(wc))(*wc)
            self._bcat = (C.c_void_p * len(bc))(*bc)
            _lib.check(self.lib.fl_set_merged_out(self.handle, self._wcat, self._bcat))
        if self.merged_in:
            wi = [self.w[f"layers.{l}.w_in"].data_ptr() for l in range(spec.n_layer)]
            bi = [self.w[f"layers.{l}.b_in"].data_ptr() if f"layers.{l}.b_in" in self.w else None
                  for l in range(spec.n_layer)]
            self._win = (C.c_void_p * len(wi))(*wi)
            self._bin = (C.c_void_p * len(bi))(*bi)
            _lib.check(self.lib.fl_set_merged_in(self.handle, self._win, self._bin,
                                                 int(self.merged_in_max_rows)))
        self.use_graphs = use_graphs
        _lib.check(self.lib.fl_configure(self.handle, int(use_graphs), 8, 0))
        if tp_size > 1 and comm_id is None:
            raise InvalidParam("tp_size > 1 needs comm_id (see tp.make_comm_id)")
        if comm_id is not None:      # NCCL path (at tp_size 1 it still runs the collectives)
            buf = C.create_string_buffer(bytes(comm_id), 128)
            _lib.check(self.lib.fl_comm_init(self.handle, buf, tp_rank, tp_size))

        self.cs = _cuda.Stream(device=self.device)
        # overlapped preprocessing: prompts run on a side stream
        self.side_prefill = False
        self.lane = None
        self.set_prefill(prefill, prefill_slots)
        _cuda.synchronize(self.device)      # weights / pool written on the default stream

        # ---- host bookkeeping
        self.capture_logits = capture_logits
        self.vl = (spec.vocab + tp_size - 1) // tp_size
        if capture_logits:
            self.logits_buf = torch.empty((self.max_rows, self.vl), dtype=torch.float32,
                                          device=self.device)
        self.logits_log = []             # [(iteration, [rid per decode row], cpu tensor)]
        self.time_steps = time_steps
        self._events = []
        self._new = []                    # rids fused at this boundary, in order
        self._live = {}                   # rid -> dict(P, stop, slot)
        self._orphans = {}                # logical slot -> stale context length
        self._prev_had_new = False
        self._rows_layout = None
        self._rows_version = None
        self._rows = None
        self._n_rows = self._n_dec = self._n_real_dec = 0
        self._pre_passes = []
        self.iterations = 0
        self.rows_total = 0
        self.prefill_rows_total = 0
        self.decode_rows_total = 0
        self.orphan_rows_total = 0
        self.shuffles = 0
        self.moved_kv_bytes = 0
        self.shuffle_log = []             # (moves, algorithmic bytes, device ms) per shuffle
        self.seen = []
        self._ring_owner = {}             # state-ring index -> rid whose history it holds
        self.h2d_bytes = 0
        self.d2h_bytes = 0
        self.attn_ctx_rows = 0            # sum over iterations of sum_rows ctx_r
        self._live_ctx = 0                # sum over live requests of (P + gen)
        self._tail_ctx = 0
        self.attn_bytes_total = 0.0
        self.attn_bytes_profiled = 0.0
        self._fl_calls = 0
        self._profiling = False
        self.prof_every = 8
        self._orphan_ctx = 0
        self._prefill_ctx = 0
        self.clock_reduce = None          # callable(ms) -> ms agreed across TP ranks
        self._imports = []                # (staging slot, physical slot, positions, ready event)
        self._prompt_cache = {}
        self._step_ev = self._shuffle_ev = None
        self._shuffle_pending = None
        self._n_orph = 0

    def reset(self):
        """Forget host bookkeeping between independent runs (device buffers,
        weights and the KV pool are reused; request state is re-armed at
        admission)."""
        self._new, self._live, self._orphans = [], {}, {}
        self._prev_had_new = False
        self._rows_version = None
        self._rows_layout = None
        self._rows = None
        self._n_rows = self._n_dec = 0
        self._pre_passes = []
        self._live_ctx = self._orphan_ctx = self._prefill_ctx = 0
        self.seen = []
        self._ring_owner = {}
        self.logits_log = []
        self._events = []
        self._imports = []
        if self.lane is not None:
            self.lane.reset()
            if not self.side_prefill:
                self.lane.close()
                self.lane = None

    def set_prefill(self, mode: str, slots: int = 32) -> None:
        """'inline': prompts enter the admitting fused step as PREFILL rows;
        'side': they run on a side stream as soon as they arrive
        (_PrefillLane).  Switch between serves, not inside one."""
        if mode not in ("inline", "side"):
            raise InvalidParam(f"prefill must be 'inline' or 'side', got {mode!r}")
        self.side_prefill = mode == "side"
        if self.side_prefill and self.lane is None:
            self.lane = _PrefillLane(self, slots)

    # ----------------------------------------------------------------- utils
    @property
    def stream(self):
        """The executor's own (non-default) stream: CUDA graphs cannot be
        captured on the legacy default stream."""
        return self.cs

    def launches(self) -> int:
        return int(self.lib.fl_kernel_launches(self.handle))

    def instance_pool(self, k: int) -> "InstancePool":
        """K batch-1 instances on K streams (concurrent-instances baseline)."""
        if getattr(self, "_ipool", None) is None or self._ipool.k < k:
            if getattr(self, "_ipool", None) is not None:
                self._ipool.close()
            self._ipool = InstancePool(self, k)
        return self._ipool

    def close(self):
        if getattr(self, "_ipool", None) is not None:
            self._ipool.close()
            self._ipool = None
        if getattr(self, "lane", None) is not None:
            self.lane.close()
        if getattr(self, "handle", None):
            self.lib.fl_destroy(self.handle)
            self.handle = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    # ----------------------------------------------------------------- hooks
    def on_fuse(self, rid, slot, request):
        prompt = self.prompts[rid]
        P = len(prompt)
        if request is not None and P != request.input_len:
            raise InvalidParam(f"request {rid}: prompt has {P} tokens, input_len {request.input_len}")
        if request is None:
            stop = self.max_new
        elif self.eos_token is not None:
            stop = request.max_output_length        # the EOS token may end it earlier
        else:
            stop = min(request.actual_output_length, request.max_output_length)
        if P + stop - 1 > self.S:
            raise CapacityExceeded(f"request {rid} needs {P + stop - 1} positions > max_seq {self.S}")
        if stop > self.max_new:
            raise CapacityExceeded(f"request {rid} stops at {stop} > max_new_tokens {self.max_new}")
        for other in self._live:
            if other % self.R == rid % self.R:
                raise CapacityExceeded(f"state ring collision between requests {rid} and {other}")
        self._ring_owner[rid % self.R] = rid
        staged = self.lane.take(rid) if self.side_prefill else None
        self._live[rid] = {"P": P, "stop": stop, "gen": 0, "staged": staged is not None}
        if staged is not None:
            q, ev = staged
            self._imports.append((q, slot % self.C, P - 1, ev))
        self._live_ctx += P
        self._prefill_ctx += (P - 1) * P // 2
        self._new.append(rid)
        self.seen.append(rid)

    def on_evict(self, rid, slot):
        info = self._live.pop(rid)
        self._live_ctx -= info["P"] + info["gen"]
        # KV positions written: prefill 0..P-2 plus one per generated token
        self._orphans[slot] = info["P"] + info["gen"] - 1

    def _build_rows(self, layout):
        """The iteration's row table as one int32 [n, 6] array (fl_row
        layout): window rows (DECODE / ORPHAN, window order) padded to a
        bucket, then the prompt rows of newly fused requests.  Vectorised:
        the window is read once, everything else is numpy."""
        lo, n = layout.buffer_offset, layout.buffer_size
        if n > self.C:
            raise CapacityExceeded(f"live window of {n} slots exceeds the KV pool ({self.C})")
        if self._orphans:
            for s in [k for k in self._orphans if k < lo]:
                del self._orphans[s]
        slots = layout.slots
        occ = np.fromiter((-1 if sl.occupant is None else sl.occupant for sl in slots[lo:lo + n]),
                          dtype=np.int32, count=n)
        n_dec = bucket(n)
        win = np.empty((n_dec, 6), dtype=np.int32)
        win[:] = _PAD
        w = win[:n]
        w[:, 0] = np.arange(lo, lo + n, dtype=np.int64) % self.C
        w[:, 1] = occ
        w[:, 2] = -1
        w[:, 3] = -1
        orph = occ < 0
        w[:, 4] = np.where(orph, _lib.ROW_ORPHAN, _lib.ROW_DECODE)
        w[:, 5] = 0
        if orph.any():
            idx = np.nonzero(orph)[0]
            get = self._orphans.get
            w[idx, 5] = [get(lo + int(k), 1) for k in idx]
        prefill = []
        if self._new:
            pos = {int(r): k for k, r in enumerate(occ) if r >= 0} if len(self._new) > 4 else None
            for rid in self._new:
                k = pos[rid] if pos is not None else int(np.nonzero(occ == rid)[0][0])
                pr = self._prompt_np(rid)
                P = len(pr)
                w[k, 2] = P - 1
                w[k, 3] = pr[P - 1]
                if not self._live[rid]["staged"] and P > 1:   # side-stream prefill imports its KV instead
                    blk = np.empty((P - 1, 6), dtype=np.int32)
                    blk[:, 0] = w[k, 0]
                    blk[:, 1] = rid
                    blk[:, 2] = np.arange(P - 1)
                    blk[:, 3] = pr[:P - 1]
                    blk[:, 4] = _lib.ROW_PREFILL
                    blk[:, 5] = 0
                    prefill.append(blk)
        self._n_real_dec = n
        self._n_orph = int(orph.sum())
        self._orphan_ctx = int(w[orph, 5].sum()) if self._n_orph else 0
        # prompt rows beyond the iteration's row budget run first as
        # prefill-only passes (their KV lands before the decode rows read it)
        room = self.max_rows - n_dec
        if room < 0:
            raise CapacityExceeded(f"window of {n_dec} rows > max_rows {self.max_rows}")
        pre = np.concatenate(prefill) if prefill else np.empty((0, 6), dtype=np.int32)
        cut = max(0, len(pre) - room)
        head, tail = pre[:cut], pre[cut:]
        self._pre_passes = []
        for i in range(0, len(head), self.max_rows):
            self._pre_passes.append(_pad_rows(head[i:i + self.max_rows]))
        self._tail_ctx = int((tail[:, 2] + 1).sum()) if len(tail) else 0
        rows = _pad_rows(np.concatenate([win, tail])) if len(tail) else win
        if len(rows) > self.max_rows:
            rows = np.ascontiguousarray(rows[:self.max_rows])   # padding only; real rows always fit
        return rows, len(rows), n_dec

    def _prompt_np(self, rid):
        a = self._prompt_cache.get(rid)
        if a is None:
            a = self._prompt_cache[rid] = np.asarray(self.prompts[rid], dtype=np.int32)
        return a

    def run_iteration(self, stream) -> None:
        """Launch one fused iteration (stream-ordered, non-blocking).  Under
        the device clock its duration is read later with iteration_ms(), so
        the host's end-of-iteration bookkeeping overlaps the running step."""
        layout = stream.layout
        has_new = bool(self._new)
        # rows are re-uploaded when the window changes -- or when another stream's
        # layout is served (baselines interleave one layout per instance)
        changed = (has_new or self._prev_had_new or layout.version != self._rows_version
                   or layout is not self._rows_layout)
        if changed:
            self._rows, self._n_rows, self._n_dec = self._build_rows(layout)
            self._rows_p = _rows_ptr(self._rows)
            self._rows_version = layout.version
            self._rows_layout = layout
            self.h2d_bytes += self._n_rows * C.sizeof(_lib.Row)
        main_ctx = self._live_ctx + self._orphan_ctx + (self._tail_ctx if changed else 0)
        self._tail_ctx = 0
        cs = self.stream
        timed = stream.clock == "device" or self.time_steps
        if timed:
            e0 = _cuda.Event(enable_timing=True)
            e1 = _cuda.Event(enable_timing=True)
            e0.record(cs)
        logits_ptr = self.logits_buf.data_ptr() if self.capture_logits else None
        if changed and self._pre_passes:
            for chunk in self._pre_passes:
                _lib.check(self.lib.fl_step(self.handle, _rows_ptr(chunk), len(chunk), 0, 1, None,
                                            C.c_void_p(cs.cuda_stream)))
                self._account(int((chunk[:, 2] + 1).sum()), len(chunk))
                self.rows_total += len(chunk)
                self.prefill_rows_total += len(chunk)
                self.h2d_bytes += len(chunk) * C.sizeof(_lib.Row)
            self._pre_passes = []
        if self._imports:
            # prompt KV of requests prefilled on the side stream: the step
            # waits for their prefill, then copies staging -> slot first
            for _, _, _, ev in self._imports:
                cs.wait_event(ev)
            flat = (C.c_int32 * (3 * len(self._imports)))(*[v for q, d, n, _ in self._imports for v in (q, d, n)])
            _lib.check(self.lib.fl_step_import(self.handle, C.c_void_p(self.lane.kv.data_ptr()), self.lane.Q,
                                               self.lane.S, flat, len(self._imports)))
            self.h2d_bytes += 12 * len(self._imports)
        _lib.check(self.lib.fl_step(self.handle, self._rows_p, self._n_rows, self._n_dec, int(changed),
                                    logits_ptr, C.c_void_p(cs.cuda_stream)))
        if self._imports:
            done = _cuda.Event()
            done.record(cs)
            self.lane.release([q for q, _, _, _ in self._imports], done)
            self._imports = []
        if timed:
            e1.record(cs)
            if stream.clock == "device":
                self._step_ev = (e0, e1)
            else:
                self._events.append((e0, e1))
        self._account(main_ctx, self._n_rows)
        self.iterations += 1
        self.rows_total += self._n_rows
        self.prefill_rows_total += self._n_rows - self._n_dec
        self.orphan_rows_total += self._n_orph
        self.decode_rows_total += self._n_real_dec - self._n_orph
        if self.capture_logits:
            rids = self._rows[:self._n_dec, 1].tolist()
            kinds = self._rows[:self._n_dec, 4].tolist()
            with _cuda.stream(cs):
                lg = self.logits_buf[:self._n_dec].float().cpu()
            self.logits_log.append((stream.iteration_index, rids, kinds, lg))
        self._prev_had_new = has_new
        self._new = []
        for info in self._live.values():
            info["gen"] += 1
        self._live_ctx += len(self._live)

    def iteration_ms(self) -> float:
        """Device time of the last iteration launched under the device clock
        (waits for it; agreed across TP ranks when clock_reduce is set)."""
        e0, e1 = self._step_ev
        e1.synchronize()
        ms = e0.elapsed_time(e1)
        return self.clock_reduce(ms) if self.clock_reduce else ms

    def shuffle_ms(self) -> float:
        """Device time of the last shuffle boundary (K10, or planner + K10)."""
        e0, e1 = self._shuffle_ev
        e1.synchronize()
        ms = e0.elapsed_time(e1)
        if self._shuffle_pending is not None:
            n, nbytes = self._shuffle_pending
            self.shuffle_log.append((n, nbytes, ms))
            self._shuffle_pending = None
        return self.clock_reduce(ms) if self.clock_reduce else ms

    def _account(self, ctx_sum: int, n_rows: int):
        """Algorithmic HBM bytes of this fl_step's K4 launches: K and
        V over every row's context plus q in / out, for all layers."""
        es = 2 if self.dtype == "bf16" else 4
        hl = self.spec.n_head // self.tp_size
        b = self.spec.n_layer * (ctx_sum * 2 * hl * self.spec.head_dim * es
                                 + n_rows * 2 * hl * self.spec.head_dim * es)
        self.attn_ctx_rows += ctx_sum
        self.attn_bytes_total += b
        if self._profiling and self._fl_calls % self.prof_every == 0:
            self.attn_bytes_profiled += b
        self._fl_calls += 1

    def on_shuffle(self, plan, timed: bool = False) -> None:
        """apply_shuffle on the device: the plan's moves -> K10 (launched, not
        waited for; ``timed``: bracket it for shuffle_ms())."""
        moves = []
        nbytes = 0
        for m in plan.moves:
            info = self._live[m.request_id]
            ctx = info["P"] + info["gen"] - 1      # KV positions written so far
            moves.append((m.src_slot % self.C, m.dst_slot % self.C, ctx))
            nbytes += 2 * ctx * self.spec.kv_bytes_per_token(
                2 if self.dtype == "bf16" else 4, self.tp_size)
        self.moved_kv_bytes += nbytes
        flat = (C.c_int32 * (3 * len(moves)))(*[v for mv in moves for v in mv])
        self.h2d_bytes += 12 * len(moves)
        cs = self.stream
        if timed:
            e0, e1 = _cuda.Event(enable_timing=True), _cuda.Event(enable_timing=True)
            e0.record(cs)
        _lib.check(self.lib.fl_shuffle(self.handle, flat, len(moves), C.c_void_p(cs.cuda_stream)))
        if timed:
            e1.record(cs)
            self._shuffle_ev = (e0, e1)
            self._shuffle_pending = (len(moves), nbytes)
        self.shuffles += 1
        for s in [m.src_slot for m in plan.moves]:
            self._orphans.pop(s, None)

    def eos_hits(self) -> list:
        """Live requests whose token of the iteration just run is the EOS
        token: one pinned read of the per-request next-token array after the
        step (the stop now depends on device data, so this is the one D2H
        per iteration EOS mode needs)."""
        if self.eos_token is None or not self._live:
            return []
        if self._tok_host is None:
            self._tok_host = torch.empty(self.R, dtype=torch.int32, pin_memory=self.device.type == "cuda")
        cs = self.stream
        with _cuda.stream(cs):
            self._tok_host.copy_(self.req_tok, non_blocking=True)
        cs.synchronize()
        self.d2h_bytes_eos = getattr(self, "d2h_bytes_eos", 0) + 4 * self.R
        t = self._tok_host
        R, eos = self.R, self.eos_token
        return [rid for rid in self._live if int(t[rid % R]) == eos]

    def launch_prefill(self, requests, now: float) -> int:
        """Start the prompts of ``requests`` (arrived by ``now``) on the side
        stream; returns how many were launched (the lane has a bounded number
        of staging slots; the rest wait for the next boundary)."""
        return self.lane.launch(requests, now)

    def poll_prefill(self, block: bool = False) -> list:
        """[(rid, ready time)] of side-stream prefills that completed: ready =
        the boundary they were launched at + their measured device time."""
        return self.lane.poll(block)

    def shuffle_on_device(self, layout):
        """A shuffle boundary planned AND executed on the device (SURVEY 8f #3,
        ``device_plan=True``): the window's occupancy goes up once, Alg. 1 +
        plan_shuffle run in csrc/planner.cu and K10 copies from the device
        move list (fl_shuffle_planned); the host planner is not called.  The
        plan comes back through a pinned buffer only so the host can mirror
        the layout (its next rows and evictions depend on it).  Returns
        (ShufflePlan, device ms or None)."""
        from .buffer import ShuffleMove, ShufflePlan
        lo, n = layout.buffer_offset, layout.buffer_size
        if n > self.C:
            raise CapacityExceeded(f"live window of {n} slots exceeds the KV pool ({self.C})")
        slots = layout.slots
        occ, size, ctx = [], [], []
        for s in range(lo, lo + n):
            rid = slots[s].occupant
            occ.append(0 if rid is None else 1)
            size.append(slots[s].size)
            info = self._live.get(rid) if rid is not None else None
            ctx.append(info["P"] + info["gen"] - 1 if info else 0)
        if self._plan_host is None:
            self._plan_host = torch.empty(3 + 2 * max(self.C, 1), dtype=torch.int32, pin_memory=self.device.type == "cuda")
            self._plan_bytes = torch.empty(1, dtype=torch.int64, pin_memory=self.device.type == "cuda")
        a_occ = (C.c_int32 * max(n, 1))(*occ)
        a_size = (C.c_int64 * max(n, 1))(*size)
        a_ctx = (C.c_int32 * max(n, 1))(*ctx)
        cs = self.stream
        e0, e1 = _cuda.Event(enable_timing=True), _cuda.Event(enable_timing=True)
        e0.record(cs)
        _lib.check(self.lib.fl_shuffle_planned(self.handle, a_occ, a_size, a_ctx, n, lo,
                                               C.c_void_p(self._plan_host.data_ptr()),
                                               C.c_void_p(self._plan_bytes.data_ptr()), C.c_void_p(cs.cuda_stream)))
        e1.record(cs)
        self._shuffle_ev = (e0, e1)
        self.h2d_bytes += 16 * n
        self.d2h_bytes_plans = getattr(self, "d2h_bytes_plans", 0) + 4 * (3 + 2 * n) + 8
        self.device_plans += 1
        e1.synchronize()                 # the plan read-back (ordered before e1) has landed
        out = self._plan_host
        offset, wlen, nm = int(out[0]), int(out[1]), int(out[2])
        moves = tuple(ShuffleMove(slots[int(out[3 + 2 * r])].occupant, int(out[3 + 2 * r]), int(out[4 + 2 * r]),
                                  slots[int(out[3 + 2 * r])].size) for r in range(nm))
        plan = ShufflePlan(moves, offset, wlen, int(self._plan_bytes[0]), layout.version)
        if moves:
            nbytes = 0
            for m in moves:
                info = self._live[m.request_id]
                nbytes += 2 * (info["P"] + info["gen"] - 1) * self.spec.kv_bytes_per_token(
                    2 if self.dtype == "bf16" else 4, self.tp_size)
                self._orphans.pop(m.src_slot, None)
            self.moved_kv_bytes += nbytes
            self.shuffles += 1
            self._shuffle_pending = (len(moves), nbytes)
        else:
            self._shuffle_pending = None
        return plan

    def on_drain(self, stream):
        self.cs.synchronize()

    # ----------------------------------------------------------------- results
    def step_times_ms(self) -> list:
        self.cs.synchronize()
        return [a.elapsed_time(b) for a, b in self._events]

    def tokens(self, rids=None) -> dict:
        """rid -> generated token ids: one gather on the device, one D2H copy
        of exactly the requested histories (counted in ``d2h_bytes``)."""
        rids = list(self.seen if rids is None else rids)
        if not rids:
            return {}
        for rid in rids:
            owner = self._ring_owner.get(rid % self.R)
            if owner != rid:
                raise CapacityExceeded(f"history of request {rid} was overwritten by request {owner} "
                                       f"(state_slots {self.R}); read tokens() before the ring wraps")
        with _cuda.stream(self.cs):
            idx = torch.tensor([r % self.R for r in rids], device=self.device, dtype=torch.long)
            packed = torch.cat([self.req_ngen[idx].unsqueeze(1), self.tok_hist[idx]], dim=1).cpu()
        self.d2h_bytes = packed.numel() * 4
        return {rid: packed[i, 1:1 + int(packed[i, 0])].tolist() for i, rid in enumerate(rids)}

    def profile(self, enable: bool):
        """Live kernel timing: the library brackets launch groups with events on
        one fl_step in ``prof_every`` (counting from here); the executor keeps
        the algorithmic attention bytes of exactly those steps."""
        _lib.check(self.lib.fl_profile(self.handle, int(enable)))
        self._profiling = bool(enable)
        self._fl_calls = 0
        self.attn_bytes_profiled = 0.0

    def profile_read(self) -> dict:
        out = {}
        for name, cls in (("attention", _lib.PROF_ATTENTION), ("gemm", _lib.PROF_GEMM),
                          ("shuffle", _lib.PROF_SHUFFLE), ("step", _lib.PROF_STEP)):
            ms, n, b, f = C.c_double(), C.c_int64(), C.c_double(), C.c_double()
            _lib.check(self.lib.fl_profile_read(self.handle, cls, C.byref(ms), C.byref(n), C.byref(b),
                                                C.byref(f)))
            out[name] = {"ms": ms.value, "records": n.value, "bytes": b.value, "flops": f.value}
        return out


def _side_handle(ex: "CudaExecutor", kv, state, C_slots: int, S: int, max_rows: int, R: int, max_new: int):
    """A second library handle over ex's weights (own workspace, own pool
    descriptor) whose launches may run beside other handles' on other
    streams (fl_set_side_stream: GEMMs without cross-CTA waits).  Returns
    (handle, workspace tensor, pool descriptor)."""
    if ex.tp_size > 1:
        raise InvalidParam("side handles are single-GPU (their collectives would need their own communicator)")
    lib = ex.lib
    pdesc = _lib.PoolDesc(C_slots, S, max_rows, R, max_new, ex.pdesc.use_tensor_cores, kv.data_ptr(),
                          *[t.data_ptr() for t in state], None, 0)
    nbytes = lib.fl_workspace_bytes(C.byref(ex.mdesc), C.byref(pdesc))
    if nbytes == 0:
        _lib.check(-1)
    ws = torch.empty(nbytes, dtype=torch.uint8, device=ex.device)
    pdesc.workspace = ws.data_ptr()
    pdesc.workspace_bytes = nbytes
    h = C.c_void_p()
    _lib.check(lib.fl_create(C.byref(ex.mdesc), C.byref(pdesc), C.byref(h)))
    _lib.check(lib.fl_set_side_stream(h, 1))
    if ex.merged:
        _lib.check(lib.fl_set_merged_out(h, ex._wcat, ex._bcat))
    if ex.merged_in:
        _lib.check(lib.fl_set_merged_in(h, ex._win, ex._bin, int(ex.merged_in_max_rows)))
    _lib.check(lib.fl_configure(h, int(ex.use_graphs), 8, 0))
    return h, ws, pdesc


class _PrefillLane:
    """Overlapped preprocessing: the paper's T_pp threads
     that prepare a request's context while the fused stream
    keeps iterating; the reference models them as an independent delay
    (engine.py:6-8,24-42,69-83).

    A second library handle over the same weights runs each arrived prompt's
    PREFILL rows (n_dec = 0 steps) on a side stream into a small staging
    pool [L][Q][2][Hl][S_p][hd] (S_p = prompt length); its GEMMs avoid
    cross-CTA waits (fl_set_side_stream) so it can share the SMs with the
    serving stream.  At fusion the serving step imports the prompt KV into
    the request's slot (fl_step_import) after waiting for the prefill's
    event; the staging slot is reused once that import ran.  Prompts of a
    boundary are batched into one prefill pass (one weight read)."""

    def __init__(self, ex: CudaExecutor, slots: int):
        spec = ex.spec
        self.ex = ex
        self.lib = ex.lib
        self.Q = max(1, int(slots))
        self.S = max(2, max(len(p) for p in ex.prompts.values()) if ex.prompts else 2)
        tdt = _TORCH_DTYPE[ex.dtype]
        hl = spec.n_head // ex.tp_size
        dev = ex.device
        self.kv = torch.empty((spec.n_layer, self.Q, 2, hl, self.S, spec.head_dim), dtype=tdt, device=dev)
        i32 = dict(dtype=torch.int32, device=dev)
        self._state = [torch.zeros(1, **i32) for _ in range(3)] + [torch.zeros((1, 1), **i32)]
        self.max_rows = bucket(min(self.Q * (self.S - 1), 512))
        self.handle, self.ws, self.pdesc = _side_handle(ex, self.kv, self._state, self.Q, self.S, self.max_rows, 1, 1)
        self.ps = _cuda.Stream(device=dev)
        self.launched_rows = 0
        self.passes = 0
        self.reset()

    def reset(self):
        self.free = list(range(self.Q))
        self.free_ev = {}          # staging slot -> event after the import that last read it
        self.inflight = {}         # rid -> [slot, e0, e1, launch time, resolved]
        self.ready = {}            # rid -> (slot, e1) prefilled, not yet fused

    def launch(self, requests, now: float) -> int:
        rids = []
        for req in requests:
            if not self.free:
                break
            rids.append((req.request_id, self.free.pop(0)))
        if not rids:
            return 0
        ex = self.ex
        rows = []
        for rid, q in rids:
            pr = ex.prompts[rid]
            rows.extend((q, rid, j, pr[j], _lib.ROW_PREFILL, 0) for j in range(len(pr) - 1))
            ev = self.free_ev.pop(q, None)
            if ev is not None:
                self.ps.wait_event(ev)          # the previous occupant's import has read it
        e0 = _cuda.Event(enable_timing=True)
        e1 = _cuda.Event(enable_timing=True)
        e0.record(self.ps)
        for i in range(0, len(rows), self.max_rows):
            chunk = rows[i:i + self.max_rows]
            chunk = chunk + [_PAD] * (bucket(len(chunk)) - len(chunk))
            arr = (_lib.Row * len(chunk))(*[_lib.Row(*r) for r in chunk])
            _lib.check(self.lib.fl_step(self.handle, arr, len(chunk), 0, 1, None, C.c_void_p(self.ps.cuda_stream)))
            ex.h2d_bytes += len(chunk) * C.sizeof(_lib.Row)
            self.launched_rows += len(chunk)
            self.passes += 1
        e1.record(self.ps)
        for rid, q in rids:
            self.inflight[rid] = [q, e0, e1, now]
        return len(rids)

    def poll(self, block: bool) -> list:
        out = []
        for rid, (q, e0, e1, t) in list(self.inflight.items()):
            if not block and not e1.query():
                continue
            e1.synchronize()
            out.append((rid, t + e0.elapsed_time(e1)))
            self.ready[rid] = (q, e1)
            del self.inflight[rid]
        return out

    def take(self, rid):
        """(staging slot, event) of rid's finished or in-flight prefill, or
        None (never launched: the prompt then runs inline in the fused step)."""
        if rid in self.ready:
            return self.ready.pop(rid)
        if rid in self.inflight:
            q, _, e1, _ = self.inflight.pop(rid)
            return q, e1
        return None

    def release(self, slots, ev):
        for q in slots:
            self.free_ev[q] = ev
            self.free.append(q)

    def close(self):
        if getattr(self, "handle", None):
            self.lib.fl_destroy(self.handle)
            self.handle = None


class InstancePool:
    """Concurrent model instances on the device: the
    reference's one-instance-per-request discipline (baselines.py:130-229)
    whose contention it MODELS with contention_gamma (cost.py:112-116).
    Here every live instance is a batch-1 decoder with its own library
    handle (own workspace, no cross-CTA waits) on its own CUDA stream, over
    the shared weights and KV pool (its own slot, its own state row), so K
    live instances really share the GPU and the contention is measured."""

    def __init__(self, ex: CudaExecutor, k: int):
        self.ex = ex
        self.k = max(1, int(k))
        # the first step of an instance: an 8-row decode window + its prompt rows
        self.S_rows = bucket(8 + (max(len(p) for p in ex.prompts.values()) if ex.prompts else 8))
        state = [ex.req_tok, ex.req_pos, ex.req_ngen, ex.tok_hist]
        self.handles, self.ws, self.streams = [], [], []
        for _ in range(self.k):
            h, ws, _ = _side_handle(ex, ex.kv, state, ex.C, ex.S, self.S_rows, ex.R, ex.max_new)
            self.handles.append(h)
            self.ws.append(ws)
            self.streams.append(_cuda.Stream(device=ex.device))
        self.free = list(range(self.k))

    def step(self, i: int, rid: int, slot: int, first: bool):
        """Launch one batch-1 decode step of request rid on instance i (the
        first also runs the prompt); returns the (start, end) events."""
        ex = self.ex
        pr = ex._prompt_np(rid)
        P = len(pr)
        phys = slot % ex.C
        if first:
            rows = np.empty((P, 6), dtype=np.int32)
            rows[0] = (phys, rid, P - 1, pr[P - 1], _lib.ROW_DECODE, 0)
            if P > 1:
                rows[1:, 0] = phys
                rows[1:, 1] = rid
                rows[1:, 2] = np.arange(P - 1)
                rows[1:, 3] = pr[:P - 1]
                rows[1:, 4] = _lib.ROW_PREFILL
                rows[1:, 5] = 0
            n_dec = 1
            dec = np.empty((8, 6), dtype=np.int32)
            dec[:] = _PAD
            dec[0] = rows[0]
            rows = _pad_rows(np.concatenate([dec, rows[1:]])) if P > 1 else dec
            n_dec = 8
        else:
            rows = np.empty((8, 6), dtype=np.int32)
            rows[:] = _PAD
            rows[0] = (phys, rid, -1, -1, _lib.ROW_DECODE, 0)
            n_dec = 8
        st = self.streams[i]
        e0, e1 = _cuda.Event(enable_timing=True), _cuda.Event(enable_timing=True)
        e0.record(st)
        _lib.check(ex.lib.fl_step(self.handles[i], _rows_ptr(rows), len(rows), n_dec, 1, None,
                                  C.c_void_p(st.cuda_stream)))
        e1.record(st)
        ex.h2d_bytes += len(rows) * C.sizeof(_lib.Row)
        ex.rows_total += len(rows)
        ex.iterations += 1
        return e0, e1

    def close(self):
        for h in self.handles:
            if h:
                self.ex.lib.fl_destroy(h)
        self.handles = []
