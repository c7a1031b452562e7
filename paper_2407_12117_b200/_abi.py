"""ctypes mirror of include/memo.h and the loader for the in-tree libmemo.so.

The library is the product: there is no Python or CPU fallback.  Importing
this module on a box where ``_lib/libmemo.so`` is missing raises immediately.
"""
from __future__ import annotations

import ctypes as C
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("MEMO_LIB_PATH") or os.path.join(_HERE, "_lib", "libmemo.so")

NUM_SKELETAL = 10
SKELETAL_NAMES = (
    "layer_input", "input_norm", "q", "k", "v", "attn_out", "attn_proj",
    "post_attn_norm", "ffn_fc1", "ffn_act",
)

MEMO_OK, MEMO_ERR_INTERNAL, MEMO_ERR_INPUT, MEMO_ERR_INFEASIBLE, MEMO_ERR_HOST_MEMORY = range(5)


class ModelConfigC(C.Structure):
    _fields_ = [(n, C.c_uint64) for n in (
        "n_layers", "hidden", "ffn_hidden", "n_heads", "vocab", "batch", "seq_len",
        "dtype_bytes", "tp_degree", "sp_or_cp_degree")] + [
        ("untied_classifier", C.c_int32),
        ("skeletal_weight", C.c_double * NUM_SKELETAL)]


class HardwareConfigC(C.Structure):
    _fields_ = [("pcie_bandwidth", C.c_double), ("cpu_mem", C.c_uint64),
                ("gpu_mem", C.c_uint64), ("peak_flops", C.c_double),
                ("efficiency", C.c_double)]


class SkeletalSizesC(C.Structure):
    _fields_ = [("s_input", C.c_uint64), ("s_attn", C.c_uint64), ("s_others", C.c_uint64),
                ("total", C.c_uint64), ("component_bytes", C.c_uint64 * NUM_SKELETAL)]


class SwapPlanC(C.Structure):
    _fields_ = [("alpha", C.c_double), ("mandatory_bytes", C.c_uint64),
                ("swapped_bytes_per_layer", C.c_uint64), ("cpu_footprint", C.c_uint64),
                ("swapped_layers", C.c_uint64), ("has_mandatory_stall", C.c_int32),
                ("mandatory_stall", C.c_double)]


class TokenSplitC(C.Structure):
    _fields_ = [("swap_tokens", C.c_uint64), ("recompute_tokens", C.c_uint64)]


class ParamCountC(C.Structure):
    _fields_ = [(n, C.c_uint64) for n in
                ("embedding", "per_layer", "final_norm", "classifier", "total")]


class TimingModelC(C.Structure):
    _fields_ = [(n, C.c_double) for n in (
        "t_fwd_layer", "t_bwd_layer", "t_attn_fwd", "t_embedding_fwd", "t_embedding_bwd",
        "t_classifier_fwd", "t_classifier_bwd", "bwd_ratio")]


class ScheduleEventC(C.Structure):
    _fields_ = [("stream", C.c_int32), ("kind", C.c_int32), ("layer", C.c_int32),
                ("start", C.c_double), ("end", C.c_double)]


class SimReportC(C.Structure):
    _fields_ = [(n, C.c_double) for n in (
        "iteration_time", "compute_blocked", "forward_blocked", "offload_stream_busy",
        "prefetch_stream_busy", "tgs", "mfu")]


class GemmArgsC(C.Structure):
    _fields_ = [("M", C.c_int32), ("N", C.c_int32), ("K", C.c_int32),
                ("a", C.c_void_p), ("lda", C.c_int64), ("a_mn_major", C.c_int32),
                ("b", C.c_void_p), ("ldb", C.c_int64), ("b_mn_major", C.c_int32),
                ("epilogue", C.c_int32), ("c", C.c_void_p), ("ldc", C.c_int64),
                ("out_f32", C.c_void_p), ("resid", C.c_void_p), ("ld_f32", C.c_int64),
                ("q", C.c_void_p), ("k", C.c_void_p), ("v", C.c_void_p),
                ("hidden", C.c_int32), ("head_dim", C.c_int32),
                ("rope", C.c_void_p), ("pos0", C.c_int64), ("variant", C.c_int32),
                ("raster", C.c_int32)]


class MemoError(RuntimeError):
    def __init__(self, code: int, msg: str):
        super().__init__(f"[memo status {code}] {msg}")
        self.code = code


def _load():
    if not os.path.exists(LIB_PATH):
        raise ImportError(
            f"libmemo.so not built at {LIB_PATH}; run `python -c 'import __graft_entry__ as g; "
            "g.build()'` (the CUDA path has no fallback)")
    lib = C.CDLL(LIB_PATH)
    lib.memo_last_error.restype = C.c_char_p
    lib.memo_version.restype = C.c_char_p
    for name in ("memo_flops_per_sample", "memo_mfu_from_tgs"):
        if hasattr(lib, name):
            getattr(lib, name).restype = C.c_double
    lib.memo_attn_bwd_workspace_bytes.restype = C.c_uint64
    return lib


lib = _load()


def check(code: int) -> None:
    if code != MEMO_OK:
        raise MemoError(code, lib.memo_last_error().decode())


def take_string(p: C.c_char_p) -> str:
    """Copy and free a heap string returned by the library."""
    s = C.cast(p, C.c_char_p).value.decode()
    lib.memo_free(p)
    return s
