"""Python mirror of the reference's planning interface (proj/include/actmem),
implemented by the C++ host planner behind include/memo.h.

Names, argument meaning and error behaviour follow the reference:
``skeletal_sizes`` (swap.hpp:75), ``solve_alpha`` (swap.hpp:105),
``make_swap_plan_with_alpha`` (schedule.hpp:409), ``token_split``
(swap.hpp:177), ``count_params`` (schedule.hpp:44), ``analytic_timing``
(schedule.hpp:100), ``plan_model`` (bilevel.hpp:189), ``build_schedule``
(schedule.hpp:186), ``validate_schedule`` (:301), ``simulate`` (:260).
Reference exception classes map to MemoError codes 2/3/4.
"""
from __future__ import annotations

import ctypes as C
import json
import math
from dataclasses import dataclass, field
from typing import Dict, List, Optional

from ._abi import (NUM_SKELETAL, SKELETAL_NAMES, HardwareConfigC, MemoError, ModelConfigC,
                   ParamCountC, ScheduleEventC, SimReportC, SkeletalSizesC, SwapPlanC,
                   TimingModelC, TokenSplitC, check, lib, take_string)

KiB, MiB, GiB = 1024, 1024 ** 2, 1024 ** 3

STREAMS = ("compute", "offload", "prefetch")
KINDS = ("embedding_fwd", "layer_fwd", "classifier_fwd", "classifier_bwd", "recompute",
         "layer_bwd", "embedding_bwd", "offload", "prefetch")


@dataclass
class ModelConfig:  # types.hpp:80-123
    n_layers: int = 1
    hidden: int = 1
    ffn_hidden: int = 1
    n_heads: int = 1
    vocab: int = 1
    batch: int = 1
    seq_len: int = 1
    dtype_bytes: int = 2
    tp_degree: int = 1
    sp_or_cp_degree: int = 1
    untied_classifier: bool = False
    skeletal_weights: Dict[str, float] = field(default_factory=dict)

    def seq_local(self) -> int:
        return self.seq_len // self.sp_or_cp_degree

    def hidden_local(self) -> int:
        return self.hidden // self.tp_degree

    def model_gpus(self) -> int:
        return self.tp_degree * self.sp_or_cp_degree

    def to_c(self) -> ModelConfigC:
        c = ModelConfigC()
        for f in ("n_layers", "hidden", "ffn_hidden", "n_heads", "vocab", "batch", "seq_len",
                  "dtype_bytes", "tp_degree", "sp_or_cp_degree"):
            setattr(c, f, int(getattr(self, f)))
        c.untied_classifier = int(bool(self.untied_classifier))
        for i, name in enumerate(SKELETAL_NAMES):
            c.skeletal_weight[i] = float(self.skeletal_weights.get(name, math.nan))
        return c

    def to_json(self) -> dict:
        d = {k: getattr(self, k) for k in ("n_layers", "hidden", "ffn_hidden", "n_heads", "vocab",
                                           "batch", "seq_len", "dtype_bytes", "tp_degree",
                                           "sp_or_cp_degree", "untied_classifier")}
        if self.skeletal_weights:
            d["skeletal_weights"] = dict(self.skeletal_weights)
        return d


@dataclass
class HardwareConfig:  # types.hpp:126-141
    pcie_bandwidth: float = 32.0e9
    cpu_mem: int = 2048 * GiB
    gpu_mem: int = 80 * GiB
    peak_flops: float = 312.0e12
    efficiency: float = 0.5

    def to_c(self) -> HardwareConfigC:
        return HardwareConfigC(float(self.pcie_bandwidth), int(self.cpu_mem), int(self.gpu_mem),
                               float(self.peak_flops), float(self.efficiency))


@dataclass
class SkeletalSizes:  # swap.hpp:67-73
    s_input: int
    s_attn: int
    s_others: int
    total: int
    components: List[tuple]

    def to_c(self) -> SkeletalSizesC:
        c = SkeletalSizesC(self.s_input, self.s_attn, self.s_others, self.total)
        for i, (_, b) in enumerate(self.components[:NUM_SKELETAL]):
            c.component_bytes[i] = b
        return c


@dataclass
class SwapPlan:  # swap.hpp:94-103
    alpha: float
    mandatory_bytes: int
    swapped_bytes_per_layer: int
    cpu_footprint: int
    swapped_layers: int
    mandatory_stall: Optional[float] = None

    def to_c(self) -> SwapPlanC:
        return SwapPlanC(self.alpha, self.mandatory_bytes, self.swapped_bytes_per_layer,
                         self.cpu_footprint, self.swapped_layers,
                         int(self.mandatory_stall is not None), self.mandatory_stall or 0.0)


@dataclass
class TimingModel:  # schedule.hpp:74-95
    t_fwd_layer: float = 0.0
    t_bwd_layer: float = 0.0
    t_attn_fwd: float = 0.0
    t_embedding_fwd: float = 0.0
    t_embedding_bwd: float = 0.0
    t_classifier_fwd: float = 0.0
    t_classifier_bwd: float = 0.0
    bwd_ratio: float = 2.0

    def to_c(self) -> TimingModelC:
        return TimingModelC(self.t_fwd_layer, self.t_bwd_layer, self.t_attn_fwd,
                            self.t_embedding_fwd, self.t_embedding_bwd, self.t_classifier_fwd,
                            self.t_classifier_bwd, self.bwd_ratio)


@dataclass
class ScheduleEvent:  # schedule.hpp:162-168
    stream: str
    kind: str
    layer: int
    start: float
    end: float


def _swap_from_c(c: SwapPlanC) -> SwapPlan:
    return SwapPlan(c.alpha, c.mandatory_bytes, c.swapped_bytes_per_layer, c.cpu_footprint,
                    c.swapped_layers, c.mandatory_stall if c.has_mandatory_stall else None)


def skeletal_sizes(cfg: ModelConfig) -> SkeletalSizes:
    out = SkeletalSizesC()
    check(lib.memo_skeletal_sizes_of(C.byref(cfg.to_c()), C.byref(out)))
    comps = [(SKELETAL_NAMES[i], out.component_bytes[i]) for i in range(NUM_SKELETAL)]
    return SkeletalSizes(out.s_input, out.s_attn, out.s_others, out.total, comps)


def solve_alpha(sz: SkeletalSizes, hw: HardwareConfig, t_layer_fwd: float, n_layers: int) -> SwapPlan:
    out = SwapPlanC()
    check(lib.memo_solve_alpha(C.byref(sz.to_c()), C.byref(hw.to_c()), C.c_double(t_layer_fwd),
                               C.c_uint64(n_layers), C.byref(out)))
    return _swap_from_c(out)


def make_swap_plan_with_alpha(sz: SkeletalSizes, hw: HardwareConfig, alpha: float, n_layers: int) -> SwapPlan:
    out = SwapPlanC()
    check(lib.memo_swap_plan_with_alpha(C.byref(sz.to_c()), C.byref(hw.to_c()), C.c_double(alpha),
                                        C.c_uint64(n_layers), C.byref(out)))
    return _swap_from_c(out)


def token_split(alpha: float, seq_len_local: int, granularity: int = 128):
    out = TokenSplitC()
    check(lib.memo_token_split_of(C.c_double(alpha), C.c_uint64(seq_len_local),
                                  C.c_uint64(granularity), C.byref(out)))
    return out.swap_tokens, out.recompute_tokens


def count_params(cfg: ModelConfig) -> dict:
    out = ParamCountC()
    check(lib.memo_count_params(C.byref(cfg.to_c()), C.byref(out)))
    return {f: getattr(out, f) for f, _ in ParamCountC._fields_}


def estimate_flops_per_sample(cfg: ModelConfig, param_count: int) -> float:
    return lib.memo_flops_per_sample(C.byref(cfg.to_c()), C.c_uint64(param_count))


def mfu_from_tgs(cfg: ModelConfig, hw: HardwareConfig, param_count: int, tgs: float) -> float:
    return lib.memo_mfu_from_tgs(C.byref(cfg.to_c()), C.byref(hw.to_c()), C.c_uint64(param_count),
                                 C.c_double(tgs))


def analytic_timing(cfg: ModelConfig, hw: HardwareConfig) -> TimingModel:
    out = TimingModelC()
    check(lib.memo_analytic_timing(C.byref(cfg.to_c()), C.byref(hw.to_c()), C.byref(out)))
    return TimingModel(*[getattr(out, f) for f, _ in TimingModelC._fields_])


def plan_model_json(trace_text: str, cap: int = 0, time_budget: float = 60.0,
                    alignment: int = 512) -> str:
    """bilevel.hpp:189 plan_model; returns json_io.hpp:189 to_json(GlobalPlan).dump()."""
    p = C.c_char_p()
    check(lib.memo_plan_model(trace_text.encode(), C.c_uint64(cap), C.c_double(time_budget),
                              C.c_uint64(alignment), C.byref(p)))
    return take_string(p)


def plan_model(trace_text: str, cap: int = 0, time_budget: float = 60.0, alignment: int = 512) -> dict:
    return json.loads(plan_model_json(trace_text, cap, time_budget, alignment))


def solve_dsa(trace_text: str, cap: int = 0, time_budget: float = 60.0, alignment: int = 512) -> dict:
    p = C.c_char_p()
    check(lib.memo_solve_dsa(trace_text.encode(), C.c_uint64(cap), C.c_double(time_budget),
                             C.c_uint64(alignment), C.byref(p)))
    return json.loads(take_string(p))


def trace_roundtrip(trace_text: str) -> str:
    p = C.c_char_p()
    check(lib.memo_trace_roundtrip(trace_text.encode(), C.byref(p)))
    return take_string(p)


def _events_to_c(events):
    arr = (ScheduleEventC * max(1, len(events)))()
    for i, e in enumerate(events):
        s = STREAMS.index(e.stream) if isinstance(e.stream, str) else e.stream
        k = KINDS.index(e.kind) if isinstance(e.kind, str) else e.kind
        arr[i] = ScheduleEventC(s, k, e.layer, e.start, e.end)
    return arr


def build_schedule(cfg: ModelConfig, hw: HardwareConfig, sz: SkeletalSizes, swap: SwapPlan,
                   tm: TimingModel) -> List[ScheduleEvent]:
    n = C.c_size_t()
    args = (C.byref(cfg.to_c()), C.byref(hw.to_c()), C.byref(sz.to_c()), C.byref(swap.to_c()),
            C.byref(tm.to_c()))
    check(lib.memo_build_schedule(*args, None, C.c_size_t(0), C.byref(n)))
    arr = (ScheduleEventC * max(1, n.value))()
    check(lib.memo_build_schedule(*args, arr, C.c_size_t(n.value), C.byref(n)))
    return [ScheduleEvent(STREAMS[e.stream], KINDS[e.kind], e.layer, e.start, e.end)
            for e in arr[:n.value]]


def validate_schedule(events: List[ScheduleEvent], n_layers: int, swap: SwapPlan) -> List[str]:
    p = C.c_char_p()
    check(lib.memo_validate_schedule(_events_to_c(events), C.c_size_t(len(events)),
                                     C.c_uint64(n_layers), C.byref(swap.to_c()), C.byref(p)))
    s = take_string(p)
    return s.split("\n") if s else []


def simulate(events: List[ScheduleEvent], cfg: ModelConfig, hw: HardwareConfig, param_count: int) -> dict:
    out = SimReportC()
    check(lib.memo_simulate(_events_to_c(events), C.c_size_t(len(events)), C.byref(cfg.to_c()),
                            C.byref(hw.to_c()), C.c_uint64(param_count), C.byref(out)))
    return {f: getattr(out, f) for f, _ in SimReportC._fields_}


def schedule_timeline_csv(events: List[ScheduleEvent]) -> str:
    """json_io.hpp:246-254: `stream,kind,layer,start,end` with 17 significant digits."""
    out = ["stream,kind,layer,start,end"]
    for e in events:
        out.append(f"{e.stream},{e.kind},{e.layer},{e.start:.17g},{e.end:.17g}")
    return "\n".join(out) + "\n"


def fnv1a_hex(data: str) -> str:
    b = data.encode()
    out = C.create_string_buffer(19)
    check(lib.memo_fnv1a_hex(b, C.c_size_t(len(b)), out))
    return out.value.decode()


def load_run_config(json_text: str):
    """json_io.hpp:141-176; returns (ModelConfig, HardwareConfig, planner, swap, synth_seed)."""
    m, h = ModelConfigC(), HardwareConfigC()
    cap, align, gran, seed = C.c_uint64(), C.c_uint64(), C.c_uint64(), C.c_uint64()
    budget, t_layer = C.c_double(), C.c_double()
    check(lib.memo_parse_run_config(json_text.encode(), C.byref(m), C.byref(h), C.byref(cap),
                                    C.byref(align), C.byref(budget), C.byref(gran),
                                    C.byref(t_layer), C.byref(seed)))
    cfg = ModelConfig(*[getattr(m, f) for f in ("n_layers", "hidden", "ffn_hidden", "n_heads",
                                                "vocab", "batch", "seq_len", "dtype_bytes",
                                                "tp_degree", "sp_or_cp_degree")],
                      untied_classifier=bool(m.untied_classifier),
                      skeletal_weights={SKELETAL_NAMES[i]: m.skeletal_weight[i]
                                        for i in range(NUM_SKELETAL)
                                        if not math.isnan(m.skeletal_weight[i])})
    hw = HardwareConfig(h.pcie_bandwidth, h.cpu_mem, h.gpu_mem, h.peak_flops, h.efficiency)
    return (cfg, hw, {"cap": cap.value, "alignment": align.value, "time_budget": budget.value},
            {"token_granularity": gran.value, "t_layer": t_layer.value}, seed.value)


__all__ = ["ModelConfig", "HardwareConfig", "SkeletalSizes", "SwapPlan", "TimingModel",
           "ScheduleEvent", "MemoError", "skeletal_sizes", "solve_alpha",
           "make_swap_plan_with_alpha", "token_split", "count_params", "estimate_flops_per_sample",
           "mfu_from_tgs", "analytic_timing", "plan_model", "plan_model_json", "solve_dsa",
           "trace_roundtrip", "build_schedule", "validate_schedule", "simulate", "fnv1a_hex",
           "schedule_timeline_csv",
           "load_run_config"]
