"""Bit-exact parity of the C++ host planner (libmemo) with the reference actmem
planner, against golden vectors produced by the UNMODIFIED reference headers
(tests/golden/make_goldens.py -> oracle/_ref/ref_probe).

Covers SURVEY §8(a) rows A1-A14: skeletal bytes, alpha, token split, params,
FLOPs, analytic timing, trace round trip, DSA offsets, bi-level plan JSON (FNV
hashes and full text), schedule events, validator and simulator outputs.
"""
import gzip
import json
import math
import os

import pytest

from paper_2407_12117_b200 import planner as P
from paper_2407_12117_b200._abi import MemoError

G = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def _load(name):
    with open(os.path.join(G, name)) as f:
        return json.load(f)


def _gz(rel):
    with gzip.open(os.path.join(G, rel), "rt") as f:
        return f.read()


CONFIGS = _load("ref_configs.json")


def _model(d):
    return P.ModelConfig(**{k: v for k, v in d.items() if k != "skeletal_weights"},
                         skeletal_weights=d.get("skeletal_weights", {}))


def _hw(d):
    return P.HardwareConfig(**d)


@pytest.mark.parametrize("name", sorted(CONFIGS))
def test_config_report_parity(name):
    rec = CONFIGS[name]
    cfg, hw = _model(rec["model"]), _hw(rec["hardware"])
    sz = P.skeletal_sizes(cfg)
    assert [[n, b] for n, b in sz.components] == rec["skeletal"]["components"]
    assert (sz.s_input, sz.s_attn, sz.s_others, sz.total) == (
        rec["skeletal"]["s_input"], rec["skeletal"]["s_attn"], rec["skeletal"]["s_others"],
        rec["skeletal"]["total"])
    params = P.count_params(cfg)
    for k in ("embedding", "per_layer", "final_norm", "classifier", "total"):
        assert params[k] == rec["params"][k]
    assert P.estimate_flops_per_sample(cfg, params["total"]) == rec["flops_per_sample"]
    tm = P.analytic_timing(cfg, hw)
    for k, v in rec["timing"].items():
        assert getattr(tm, k) == v, k
    if "swap_error" in rec:
        with pytest.raises(MemoError) as ei:
            P.solve_alpha(sz, hw, tm.t_fwd_layer, cfg.n_layers)
        assert ei.value.code == 4
    elif "swap" in rec:
        sw = rec["swap"]
        # forced alphas (cfg1, cfg5 sweep) use make_swap_plan_with_alpha; others solve_alpha
        forced = name.startswith("cfg1") or name.startswith("cfg5")
        plan = (P.make_swap_plan_with_alpha(sz, hw, sw["alpha"], cfg.n_layers) if forced
                else P.solve_alpha(sz, hw, tm.t_fwd_layer, cfg.n_layers))
        assert plan.alpha == sw["alpha"]
        assert plan.mandatory_bytes == sw["mandatory_bytes"]
        assert plan.swapped_bytes_per_layer == sw["swapped_bytes_per_layer"]
        assert plan.cpu_footprint == sw["cpu_footprint"]
        assert plan.swapped_layers == sw["swapped_layers"]
        stall = sw["blocking"]["stall_seconds"] if sw["blocking"] else None
        assert plan.mandatory_stall == stall
        st, rc = P.token_split(plan.alpha, cfg.seq_local(), 128)
        assert (st, rc) == (rec["token_split"]["swap_tokens"], rec["token_split"]["recompute_tokens"])
        events = P.build_schedule(cfg, hw, sz, plan, tm)
        ref_ev = rec["schedule_events"]
        assert len(events) == len(ref_ev)
        for e, r in zip(events, ref_ev):
            assert (P.STREAMS.index(e.stream), P.KINDS.index(e.kind), e.layer, e.start, e.end) == tuple(r)
        assert P.validate_schedule(events, cfg.n_layers, plan) == rec["schedule_violations"]
        sim = P.simulate(events, cfg, hw, params["total"])
        for k, v in rec["sim"].items():
            assert sim[k] == v, k


@pytest.mark.parametrize("name", sorted(k for k, v in CONFIGS.items() if "trace_text_file" in v))
def test_config_plan_bit_exact(name):
    rec = CONFIGS[name]
    text = _gz(rec["trace_text_file"])
    assert P.fnv1a_hex(text) == rec["trace_fnv"]
    assert P.trace_roundtrip(text) == text
    pj = P.plan_model_json(text, 0, 60.0, 512)
    assert P.fnv1a_hex(pj) == rec["plan_fnv"]
    assert pj == _gz(rec["plan_json_file"])
    plan = json.loads(pj)
    assert plan["total_peak"] == rec["total_peak"]
    assert plan["optimal"] is True


def test_survey_goldens():
    # SURVEY §8c survey-computed hashes (cfg1, cfg1', cfg2, cfg3).
    want = {"cfg1": ("0x0216d7360a4e72ff", "0x578911ad44a4cd64"),
            "cfg1p": ("0xe611d2309a15b8a3", "0x71bdf83e5d5179a5"),
            "cfg2": ("0x33fa97058d8bf8df", "0xa03037efbb6fe797"),
            "cfg3": ("0x06881f08c6351a7f", "0xfad42307c3e8be14")}
    for name, (t, p) in want.items():
        assert CONFIGS[name]["trace_fnv"] == t and CONFIGS[name]["plan_fnv"] == p


RANDOM_PLANS = _load("ref_random_plans.json")


@pytest.mark.parametrize("i", range(len(RANDOM_PLANS)))
def test_random_iteration_plans(i):
    case = RANDOM_PLANS[i]
    pj = P.plan_model_json(case["trace"], 0, 30.0, case["alignment"])
    assert pj == case["plan_json"]


DSA = _load("ref_dsa.json")


@pytest.mark.parametrize("i", range(len(DSA)))
def test_dsa_exact_and_heuristic(i):
    case = DSA[i]
    r = P.solve_dsa(case["trace"], 0, 10.0, case["alignment"])
    assert r["lower_bound"] == case["lower_bound"]
    assert r["status"] == case["exact"]["status"]
    assert r["peak"] == case["exact"]["peak"] == case["oracle_peak"]
    assert r["addresses"] == case["exact"]["addresses"]
    assert r["heuristic"]["addresses"] == case["heuristic"]["addresses"]
    assert r["heuristic"]["peak"] == case["heuristic"]["peak"]
    assert r["verify"] == ""


SWAP = _load("ref_swap.json")


@pytest.mark.parametrize("i", range(len(SWAP["solve_alpha"])))
def test_solve_alpha_goldens(i):
    c = SWAP["solve_alpha"][i]
    si, sa, so, tot = c["sz"]
    sz = P.SkeletalSizes(si, sa, so, tot, [])
    hw = _hw(c["hw"])
    if "error" in c:
        with pytest.raises(MemoError) as ei:
            P.solve_alpha(sz, hw, c["t_layer"], c["n_layers"])
        assert ei.value.code == 4
        return
    plan = P.solve_alpha(sz, hw, c["t_layer"], c["n_layers"])
    ref = c["plan"]
    assert plan.alpha == ref["alpha"]
    assert plan.swapped_bytes_per_layer == ref["swapped_bytes_per_layer"]
    assert plan.cpu_footprint == ref["cpu_footprint"]
    assert plan.mandatory_stall == (ref["blocking"]["stall_seconds"] if ref["blocking"] else None)


def test_token_split_goldens():
    for a, s, g, sw, rc in SWAP["token_split"]:
        assert P.token_split(a, s, g) == (sw, rc)
    # test_swap.cpp:233-249
    assert P.token_split(0.75, 1024, 128) == (768, 256)
    assert P.token_split(0.5, 1000, 128) == (384, 616)
    assert P.token_split(1.0, 1000, 128) == (1000, 0)
    with pytest.raises(MemoError) as ei:
        P.token_split(1.5, 100)
    assert ei.value.code == 2


SCHED = _load("ref_schedule.json")


@pytest.mark.parametrize("i", range(len(SCHED)))
def test_schedule_goldens(i):
    c = SCHED[i]
    cfg, hw = _model(c["model"]), _hw(c["hardware"])
    sz = P.SkeletalSizes(0, 0, 0, c["sz_total"], [])
    sw = c["swap"]
    swap = P.SwapPlan(sw["alpha"], sw["mandatory_bytes"], sw["swapped_bytes_per_layer"],
                      sw["cpu_footprint"], sw["swapped_layers"])
    tm = P.TimingModel(**c["timing"])
    events = P.build_schedule(cfg, hw, sz, swap, tm)
    assert [[P.STREAMS.index(e.stream), P.KINDS.index(e.kind), e.layer, e.start, e.end]
            for e in events] == c["events"]
    assert P.validate_schedule(events, cfg.n_layers, swap) == c["violations"]
    assert P.schedule_timeline_csv(events) == c["timeline_csv"]  # json_io.hpp:246
    sim = P.simulate(events, cfg, hw, c["params"])
    for k, v in c["sim"].items():
        assert sim[k] == v


def test_known_answers_from_reference_tests():
    # test_swap.cpp:63-71 — 1M-token 7B skeletal bytes.
    cfg = P.ModelConfig(n_layers=32, hidden=4096, ffn_hidden=16384, n_heads=32, vocab=50257,
                        batch=1, seq_len=1 << 20, dtype_bytes=2)
    sz = P.skeletal_sizes(cfg)
    assert sz.total == 128 * P.GiB and sz.s_attn == 8 * P.GiB and sz.s_input == 16 * P.GiB
    # test_schedule.cpp:81-94 — parameter counts.
    c7 = P.ModelConfig(n_layers=32, hidden=4096, ffn_hidden=16384, n_heads=32, vocab=50257,
                       seq_len=4096)
    p = P.count_params(c7)
    assert p["embedding"] == 205852672 and p["per_layer"] == 201342976 and p["total"] == 6648836096
    c7.untied_classifier = True
    assert P.count_params(c7)["total"] == 6854688768
    # test_schedule.cpp:114-123 — MFU cross-check (A800 peak 312 TF).
    c7.untied_classifier = False
    hw = P.HardwareConfig()
    mfu = P.mfu_from_tgs(c7, hw, 6648836096, 3578.86)
    assert abs(mfu - 0.4945) < 0.4945 * 0.021
    # test_swap.cpp:106-122 — alpha worked instance 5/13.
    sz2 = P.SkeletalSizes(2_000_000_000, 1_000_000_000, 13_000_000_000, 16_000_000_000, [])
    plan = P.solve_alpha(sz2, P.HardwareConfig(pcie_bandwidth=1e9, cpu_mem=1 << 60), 8.0, 32)
    assert abs(plan.alpha - 5.0 / 13.0) < 1e-12


def test_error_codes():
    with pytest.raises(MemoError) as ei:
        P.plan_model_json("malloc 1 10\n")
    assert ei.value.code == 2  # event before segment header -> TraceParseError
    with pytest.raises(MemoError) as ei:
        P.plan_model_json("# segment layer_fwd 0\nmalloc 1 8\nfree 1 8\n")
    assert ei.value.code == 3  # wrong iteration structure -> PlanningError
    text = _gz(CONFIGS["cfg1"]["trace_text_file"])
    with pytest.raises(MemoError) as ei:
        P.plan_model_json(text, cap=1024)
    assert ei.value.code == 3  # InfeasibleError
    with pytest.raises(MemoError) as ei:
        P.load_run_config('{"model": {"n_layerz": 3}}')
    assert ei.value.code == 2


def test_load_run_config_reference_files():
    toy = json.dumps({"model": {"n_layers": 4, "hidden": 64, "ffn_hidden": 256, "n_heads": 4,
                                "vocab": 512, "batch": 1, "seq_len": 1024, "dtype_bytes": 2,
                                "tp_degree": 1, "sp_or_cp_degree": 1},
                      "hardware": {"pcie_bandwidth": 32e9, "cpu_mem": 2199023255552,
                                   "gpu_mem": 85899345920, "peak_flops": 312e12,
                                   "efficiency": 0.5},
                      "synth": {"seed": 0},
                      "planner": {"cap": 0, "alignment": 512, "time_budget": 30.0},
                      "swap": {"token_granularity": 128}})
    cfg, hw, planner, swap, seed = P.load_run_config(toy)
    assert cfg.n_layers == 4 and cfg.hidden == 64 and hw.cpu_mem == 2199023255552
    assert planner["time_budget"] == 30.0 and swap["token_granularity"] == 128
    assert cfg.to_json() == {k: v for k, v in CONFIGS["ref_toy"]["model"].items()}
