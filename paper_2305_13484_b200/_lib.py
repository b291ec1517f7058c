"""ctypes binding of the C-ABI in include/flover_b200.h.

The library is loaded from the package directory (built in-tree by
build.py).  There is no fallback: if the shared object is missing or does
not export the ABI, importing the device path raises.
"""

from __future__ import annotations

import ctypes as C
import os

from .errors import DeviceError, raise_for_status

# FL_LIB: an alternative build of the same library (A/B timing in tools/)
LIB_PATH = os.environ.get("FL_LIB") or os.path.join(os.path.dirname(os.path.abspath(__file__)),
                                                    "libflover_b200.so")

FL_FAMILY = {"gpt2": 0, "gptj": 1, "neox": 2}
FL_DTYPE = {"f32": 0, "bf16": 1}
ROW_DECODE, ROW_PREFILL, ROW_ORPHAN = 0, 1, 2
W_LAYER_COUNT = 12
EXPORTS = ("fl_abi_version", "fl_last_error", "fl_workspace_bytes", "fl_create", "fl_destroy",
           "fl_comm_unique_id", "fl_comm_init", "fl_step", "fl_shuffle", "fl_kernel_launches",
           "fl_gemm_workspace_bytes", "fl_gemm", "fl_profile", "fl_profile_read", "fl_configure",
           "fl_last_duration_ms", "fl_attention_workspace_bytes", "fl_attention",
           "fl_gemm_debug", "fl_attention_debug", "fl_plan_shuffle", "fl_tiled_weight_bytes", "fl_tile_weight",
           "fl_set_merged_out", "fl_set_merged_in", "fl_gemm2", "fl_gemm_set_rearm", "fl_gemm_tune",
           "fl_set_side_stream", "fl_step_import", "fl_shuffle_planned")
PROF_ATTENTION, PROF_GEMM, PROF_SHUFFLE, PROF_STEP = 0, 1, 2, 3


class ModelDesc(C.Structure):
    _fields_ = [("family", C.c_int32), ("dtype", C.c_int32), ("n_layer", C.c_int32),
                ("d_model", C.c_int32), ("n_head", C.c_int32), ("head_dim", C.c_int32),
                ("d_ff", C.c_int32), ("vocab", C.c_int32), ("max_pos", C.c_int32),
                ("rotary_dim", C.c_int32), ("ln_eps", C.c_float), ("tp_rank", C.c_int32),
                ("tp_size", C.c_int32), ("wte", C.c_void_p), ("wpe", C.c_void_p),
                ("lnf_g", C.c_void_p), ("lnf_b", C.c_void_p), ("w_lm", C.c_void_p),
                ("b_lm", C.c_void_p), ("layers", C.POINTER(C.c_void_p))]


class PoolDesc(C.Structure):
    _fields_ = [("pool_slots", C.c_int32), ("max_seq", C.c_int32), ("max_rows", C.c_int32),
                ("state_slots", C.c_int32), ("max_new_tokens", C.c_int32),
                ("use_tensor_cores", C.c_int32), ("kv", C.c_void_p),
                ("req_tok", C.c_void_p), ("req_pos", C.c_void_p), ("req_ngen", C.c_void_p),
                ("tok_hist", C.c_void_p), ("workspace", C.c_void_p),
                ("workspace_bytes", C.c_size_t)]


class Row(C.Structure):
    _fields_ = [("slot", C.c_int32), ("rid", C.c_int32), ("pos", C.c_int32), ("tok", C.c_int32),
                ("kind", C.c_int32), ("ctx", C.c_int32)]


_lib = None


def load() -> C.CDLL:
    """Load the in-tree .so (raises if absent -- no CPU fallback exists)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise DeviceError(f"{LIB_PATH} missing: build it with `python -m paper_2305_13484_b200.build`")
    lib = C.CDLL(LIB_PATH, mode=C.RTLD_GLOBAL)
    for name in EXPORTS:
        if not hasattr(lib, name):
            raise DeviceError(f"{LIB_PATH} does not export {name}")
    lib.fl_abi_version.restype = C.c_int
    lib.fl_last_error.restype = C.c_char_p
    lib.fl_workspace_bytes.restype = C.c_size_t
    lib.fl_workspace_bytes.argtypes = [C.POINTER(ModelDesc), C.POINTER(PoolDesc)]
    lib.fl_create.argtypes = [C.POINTER(ModelDesc), C.POINTER(PoolDesc), C.POINTER(C.c_void_p)]
    lib.fl_destroy.argtypes = [C.c_void_p]
    lib.fl_comm_unique_id.argtypes = [C.c_void_p]
    lib.fl_comm_init.argtypes = [C.c_void_p, C.c_void_p, C.c_int, C.c_int]
    lib.fl_step.argtypes = [C.c_void_p, C.POINTER(Row), C.c_int, C.c_int, C.c_int, C.c_void_p,
                            C.c_void_p]
    lib.fl_shuffle.argtypes = [C.c_void_p, C.POINTER(C.c_int32), C.c_int, C.c_void_p]
    lib.fl_kernel_launches.restype = C.c_int64
    lib.fl_kernel_launches.argtypes = [C.c_void_p]
    lib.fl_gemm_workspace_bytes.restype = C.c_size_t
    lib.fl_gemm.argtypes = [C.c_void_p, C.c_int, C.c_void_p, C.c_void_p, C.c_void_p, C.c_int,
                            C.c_int, C.c_int, C.c_int, C.c_int, C.c_int, C.c_int, C.c_void_p,
                            C.c_void_p]
    lib.fl_gemm2.argtypes = [C.c_void_p, C.c_void_p, C.c_int, C.c_void_p, C.c_void_p, C.c_void_p,
                             C.c_int, C.c_int, C.c_int, C.c_int, C.c_int, C.c_int, C.c_int,
                             C.c_int, C.c_int, C.c_void_p, C.c_int, C.c_void_p, C.c_void_p]
    lib.fl_gemm_set_rearm.argtypes = [C.c_int]
    lib.fl_gemm_set_rearm.restype = None
    lib.fl_gemm_tune.argtypes = [C.c_int, C.c_int]
    lib.fl_gemm_tune.restype = None
    lib.fl_profile.argtypes = [C.c_void_p, C.c_int]
    lib.fl_configure.argtypes = [C.c_void_p, C.c_int, C.c_int, C.c_int]
    lib.fl_last_duration_ms.argtypes = [C.c_void_p, C.POINTER(C.c_float)]
    lib.fl_profile_read.argtypes = [C.c_void_p, C.c_int, C.POINTER(C.c_double),
                                    C.POINTER(C.c_int64), C.POINTER(C.c_double),
                                    C.POINTER(C.c_double)]
    lib.fl_gemm_debug.argtypes = [C.c_void_p]
    lib.fl_gemm_debug.restype = None
    lib.fl_attention_debug.argtypes = [C.c_void_p]
    lib.fl_attention_debug.restype = None
    lib.fl_attention_workspace_bytes.restype = C.c_size_t
    lib.fl_attention_workspace_bytes.argtypes = [C.c_int, C.c_int, C.c_int, C.c_int]
    lib.fl_attention.argtypes = [C.c_void_p, C.c_void_p, C.c_void_p, C.c_int, C.c_int, C.c_int,
                                 C.c_void_p, C.c_int, C.c_int, C.c_void_p, C.c_void_p, C.c_int,
                                 C.c_void_p]
    lib.fl_set_merged_out.argtypes = [C.c_void_p, C.c_void_p, C.c_void_p]
    lib.fl_set_merged_in.argtypes = [C.c_void_p, C.c_void_p, C.c_void_p, C.c_int]
    lib.fl_tiled_weight_bytes.restype = C.c_size_t
    lib.fl_tiled_weight_bytes.argtypes = [C.c_int, C.c_int]
    lib.fl_tile_weight.argtypes = [C.c_void_p, C.c_int, C.c_int, C.c_void_p, C.c_void_p]
    lib.fl_plan_shuffle.argtypes = [C.c_void_p, C.c_void_p, C.c_int, C.c_int, C.c_void_p, C.c_void_p,
                                    C.c_void_p]
    lib.fl_set_side_stream.argtypes = [C.c_void_p, C.c_int]
    lib.fl_step_import.argtypes = [C.c_void_p, C.c_void_p, C.c_int, C.c_int, C.POINTER(C.c_int32), C.c_int]
    lib.fl_shuffle_planned.argtypes = [C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.c_int, C.c_int,
                                       C.c_void_p, C.c_void_p, C.c_void_p]
    if lib.fl_abi_version() != 1:
        raise DeviceError("ABI version mismatch")
    _lib = lib
    return lib


def check(code: int) -> None:
    if code:
        raise_for_status(code, load().fl_last_error().decode(errors="replace"))
