"""Python handle on the B200 training-step executor (include/memo.h memo_exec_*).

The executor replaces the reference's simulated schedule
(proj/include/actmem/schedule.hpp:186 build_schedule, :260 simulate) with real
execution; its measured timeline comes back in the reference's ScheduleEvent
vocabulary and is checked with the same validate_schedule / simulate.
"""
from __future__ import annotations

import ctypes as C
from typing import Optional

import numpy as np

from ._abi import SwapPlanC, TokenSplitC, SkeletalSizesC, ScheduleEventC, check, lib, take_string
from .planner import KINDS, STREAMS, HardwareConfig, ModelConfig, ScheduleEvent, SwapPlan


OP_CLASSES = ("attn_fwd", "attn_bwd_prep", "attn_bwd_dkdv", "attn_bwd_dq", "gemm")


class ExecOptionsC(C.Structure):
    _fields_ = [("seed", C.c_uint64), ("alpha", C.c_double), ("token_granularity", C.c_uint64),
                ("swap_enabled", C.c_int32), ("ce_chunk", C.c_int32), ("eps", C.c_float),
                ("rope_theta", C.c_float), ("optimizer", C.c_int32), ("lr", C.c_float),
                ("beta1", C.c_float), ("beta2", C.c_float), ("adam_eps", C.c_float),
                ("weight_decay", C.c_float), ("t_layer", C.c_double),
                ("plan_time_budget", C.c_double), ("alignment", C.c_uint64),
                ("op_timing", C.c_int32), ("dry_run", C.c_int32), ("cuda_graph", C.c_int32)]


class ExecInfoC(C.Structure):
    _fields_ = [(n, C.c_int32) for n in ("S", "h", "H", "D", "F", "V", "n_layers")] + [
        ("swap", SwapPlanC), ("split", TokenSplitC), ("skeletal", SkeletalSizesC)] + [
        (n, C.c_uint64) for n in ("arena_bytes", "rb_bytes", "device_bytes", "pinned_bytes",
                                  "state_bytes")] + [
        ("param_count", C.c_int64), ("swap_enabled", C.c_int32)] + [
        (n, C.c_double) for n in ("last_step_ms", "h2d_bytes", "d2h_bytes", "offload_bytes",
                                  "prefetch_bytes")] + [("kernel_launches", C.c_int32),
        ("op_ms", C.c_double * 5), ("op_flops", C.c_double * 5), ("op_count", C.c_int32 * 5),
        ("copy_wait_ms", C.c_double)]


lib.memo_comm_loopback_group.restype = C.c_void_p
lib.memo_comm_loopback_group.argtypes = [C.c_int32]
lib.memo_comm_loopback_group_destroy.argtypes = [C.c_void_p]
lib.memo_exec_stream.restype = C.c_void_p
lib.memo_exec_stream.argtypes = [C.c_void_p]
lib.memo_exec_destroy.argtypes = [C.c_void_p]
lib.memo_exec_peer_handle.argtypes = [C.c_void_p, C.c_void_p, C.c_size_t, C.POINTER(C.c_size_t)]
lib.memo_exec_peer_connect.argtypes = [C.c_void_p, C.c_char_p, C.c_size_t]
lib.memo_exec_peer_flags.argtypes = [C.c_void_p, C.POINTER(C.c_uint64), C.c_size_t, C.POINTER(C.c_size_t)]


def default_options() -> ExecOptionsC:
    o = ExecOptionsC()
    check(lib.memo_exec_options_default(C.byref(o)))
    return o


class Executor:
    """One B200 training-step context (arena, rounding buffers, copy streams)."""

    def __init__(self, cfg: ModelConfig, hw: HardwareConfig, tp=None, **options):
        """tp: None (single GPU) or (kind, handle, rank); cfg.tp_degree is the group size.
        kind 0 (KIND_LOOPBACK) = LoopbackGroup, 1 (KIND_NCCL) = 128-byte NCCL unique id,
        2 (KIND_IPC) = peer memory over CUDA IPC (handle None; then exchange
        peer_handle() bytes and call peer_connect), 3 (KIND_PEER_LOCAL) = peer
        memory between the threads of a LoopbackGroup on one GPU."""
        o = default_options()
        for k, v in options.items():
            if not hasattr(o, k):
                raise TypeError(f"unknown executor option {k}")
            setattr(o, k, v)
        self._h = C.c_void_p()
        self.cfg = cfg
        if tp is None:
            check(lib.memo_exec_create(C.byref(cfg.to_c()), C.byref(hw.to_c()), C.byref(o),
                                       C.byref(self._h)))
        else:
            kind, handle, rank = tp
            if isinstance(handle, LoopbackGroup):
                h = handle.ptr
            elif handle is None:
                h = None
            else:
                h = C.c_char_p(bytes(handle))
            check(lib.memo_exec_create_tp(C.byref(cfg.to_c()), C.byref(hw.to_c()), C.byref(o),
                                          kind, h, rank, C.byref(self._h)))

    def peer_handle(self) -> bytes:
        """This rank's CUDA IPC handle bytes (kind 2)."""
        n = C.c_size_t()
        buf = (C.c_uint8 * 512)()
        check(lib.memo_exec_peer_handle(self._h, buf, C.c_size_t(512), C.byref(n)))
        return bytes(buf[:n.value])

    def peer_connect(self, handles) -> None:
        """Map every rank's allocation (handles in rank order, kind 2)."""
        blob = b"".join(handles)
        check(lib.memo_exec_peer_connect(self._h, C.c_char_p(blob), C.c_size_t(len(blob))))

    def peer_flags(self):
        """This rank's IPC signal flag page: signal counts per [channel][source rank] (kind 2)."""
        buf = (C.c_uint64 * 64)()
        n = C.c_size_t()
        check(lib.memo_exec_peer_flags(self._h, buf, C.c_size_t(64), C.byref(n)))
        return [int(buf[i]) for i in range(n.value)]

    def close(self):
        if self._h:
            lib.memo_exec_destroy(self._h)
            self._h = C.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:  # noqa: BLE001
            pass

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.close()

    # ------------------------------------------------------------ steps
    @staticmethod
    def _i32(a):
        a = np.ascontiguousarray(a, dtype=np.int32)
        return a, a.ctypes.data_as(C.POINTER(C.c_int32))

    def step(self, tokens, labels) -> float:
        t, tp = self._i32(tokens)
        l, lp = self._i32(labels)
        loss = C.c_float()
        check(lib.memo_exec_step(self._h, tp, lp, C.byref(loss)))
        return loss.value

    def load_batch(self, tokens, labels):
        t, tp = self._i32(tokens)
        l, lp = self._i32(labels)
        check(lib.memo_exec_load_batch(self._h, tp, lp))

    def step_resident(self):
        check(lib.memo_exec_step_resident(self._h))

    def loss(self) -> float:
        v = C.c_float()
        check(lib.memo_exec_loss(self._h, C.byref(v)))
        return v.value

    @property
    def stream(self) -> int:
        return lib.memo_exec_stream(self._h)

    # ------------------------------------------------------------ introspection
    def timeline(self):
        n = C.c_size_t()
        check(lib.memo_exec_timeline(self._h, None, C.c_size_t(0), C.byref(n)))
        arr = (ScheduleEventC * max(1, n.value))()
        check(lib.memo_exec_timeline(self._h, arr, C.c_size_t(n.value), C.byref(n)))
        return [ScheduleEvent(STREAMS[e.stream], KINDS[e.kind], e.layer, e.start, e.end)
                for e in arr[:n.value]]

    def info(self) -> dict:
        i = ExecInfoC()
        check(lib.memo_exec_get_info(self._h, C.byref(i)))
        out = {f: getattr(i, f) for f, _ in ExecInfoC._fields_
               if f not in ("swap", "split", "skeletal", "op_ms", "op_flops", "op_count")}
        out["ops"] = {name: {"ms": i.op_ms[k], "flops": i.op_flops[k], "count": i.op_count[k]}
                      for k, name in enumerate(OP_CLASSES)}
        s = i.swap
        out["swap"] = SwapPlan(s.alpha, s.mandatory_bytes, s.swapped_bytes_per_layer,
                               s.cpu_footprint, s.swapped_layers,
                               s.mandatory_stall if s.has_mandatory_stall else None)
        out["split"] = (i.split.swap_tokens, i.split.recompute_tokens)
        out["skeletal_total"] = i.skeletal.total
        out["skeletal_components"] = list(i.skeletal.component_bytes)
        return out

    def trace_text(self) -> str:
        p = C.c_char_p()
        check(lib.memo_exec_trace(self._h, C.byref(p)))
        return take_string(p)

    def plan_json(self) -> str:
        p = C.c_char_p()
        check(lib.memo_exec_plan(self._h, C.byref(p)))
        return take_string(p)

    def bind_plan(self, plan_json: str) -> None:
        """Replay an external to_json(GlobalPlan) of this executor's trace
        (memo_exec_bind_plan): status 2 if it does not fit the trace or the
        step is already captured as a CUDA graph, 3 if it needs more than the
        reserved arena."""
        check(lib.memo_exec_bind_plan(self._h, plan_json.encode()))

    def tensor_ptr(self, name: str, layer: int = -1):
        ptr, n = C.c_void_p(), C.c_size_t()
        check(lib.memo_exec_tensor(self._h, name.encode(), layer, C.byref(ptr), C.byref(n)))
        return ptr.value, n.value

    def read(self, name: str, layer: int = -1, dtype=np.float32) -> np.ndarray:
        """Host copy of a named device tensor; bf16 tensors are widened to float32."""
        _, nbytes = self.tensor_ptr(name, layer)
        if dtype == "bf16":
            raw = np.empty(nbytes // 2, dtype=np.uint16)
            check(lib.memo_exec_read(self._h, name.encode(), layer, raw.ctypes.data_as(C.c_void_p),
                                     C.c_size_t(nbytes)))
            return (raw.astype(np.uint32) << 16).view(np.float32)
        out = np.empty(nbytes // np.dtype(dtype).itemsize, dtype=dtype)
        check(lib.memo_exec_read(self._h, name.encode(), layer, out.ctypes.data_as(C.c_void_p),
                                 C.c_size_t(nbytes)))
        return out


KIND_LOOPBACK, KIND_NCCL, KIND_IPC, KIND_PEER_LOCAL, KIND_SOLO = 0, 1, 2, 3, 4


class LoopbackGroup:
    """t tensor-parallel ranks sharing one GPU (one host thread per rank)."""

    def __init__(self, size: int):
        self.size = size
        self.ptr = C.c_void_p(lib.memo_comm_loopback_group(size))
        if not self.ptr:
            raise RuntimeError("could not create loopback group")

    def __del__(self):
        if getattr(self, "ptr", None):
            lib.memo_comm_loopback_group_destroy(self.ptr)
            self.ptr = None


def nccl_unique_id() -> bytes:
    buf = (C.c_uint8 * 128)()
    check(lib.memo_comm_unique_id(buf))
    return bytes(buf)


def run_ranks(size: int, fn):
    """Run fn(rank) on `size` threads (loopback SP+TP); returns results by rank."""
    import threading
    out, err = [None] * size, [None] * size

    def body(r):
        try:
            out[r] = fn(r)
        except BaseException as e:  # noqa: BLE001
            err[r] = e
    th = [threading.Thread(target=body, args=(r,)) for r in range(size)]
    for t in th:
        t.start()
    for t in th:
        t.join()
    for e in err:
        if e is not None:
            raise e
    return out
