"""Executor planning path without a GPU (dry_run): the executor's own request
trace, its bi-level arena plan (bit-exact with the reference planner run on the
same trace), alpha / token split, and the HBM budget at the BASELINE configs."""
import json
import os
import subprocess
import tempfile

import pytest

from paper_2407_12117_b200 import planner as P
from paper_2407_12117_b200._abi import MemoError
from paper_2407_12117_b200.executor import Executor

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
PROBE = os.path.join(ROOT, "oracle", "_ref", "ref_probe")
HW = P.HardwareConfig(pcie_bandwidth=50e9, cpu_mem=96 * P.GiB, gpu_mem=180 * 10 ** 9,
                      peak_flops=2.25e15, efficiency=0.5)


def llama(n, h, H, inter, V, S):
    return P.ModelConfig(n_layers=n, hidden=h, ffn_hidden=inter * 3 // 2, n_heads=H, vocab=V,
                         batch=1, seq_len=S, dtype_bytes=2, untied_classifier=True)


CONFIGS = {
    "cfg1p": (llama(4, 256, 4, 768, 512, 4096), 0.5),
    "cfg2": (llama(4, 4096, 32, 11008, 32000, 131072), -1.0),
    "cfg5": (llama(32, 4096, 32, 11008, 32000, 262144), 0.5),
    "13b_512k": (llama(40, 5120, 40, 13824, 32000, 524288), 0.25),
}


def _ref_plan(trace):
    with tempfile.NamedTemporaryFile("w", suffix=".trace", delete=False) as f:
        f.write(trace)
    try:
        return subprocess.check_output([PROBE, "plan", f.name, "0", "60", "512"], text=True).strip()
    finally:
        os.unlink(f.name)


@pytest.mark.parametrize("name", sorted(CONFIGS))
def test_executor_trace_plan_bit_exact(name):
    cfg, alpha = CONFIGS[name]
    hw = P.HardwareConfig(**{**HW.__dict__, "cpu_mem": 2048 * P.GiB})
    ex = Executor(cfg, hw, alpha=alpha, dry_run=1)
    trace, plan = ex.trace_text(), ex.plan_json()
    info = ex.info()
    assert P.plan_model_json(trace, 0, 60.0, 512) == plan
    if os.path.exists(PROBE):
        assert _ref_plan(trace) == plan
    jp = json.loads(plan)
    assert jp["optimal"] is True and info["arena_bytes"] == jp["total_peak"]
    # rounding buffers hold exactly the skeletal model's bytes (swap.hpp:75)
    assert info["rb_bytes"] == info["skeletal_total"]
    # token split follows swap.hpp:177 at the executor's alpha
    st, rc = P.token_split(info["swap"].alpha, cfg.seq_len, 128)
    assert info["split"] == (st, rc)


def test_cfg2_fits_one_b200():
    cfg, _ = CONFIGS["cfg2"]
    ex = Executor(cfg, HW, dry_run=1)
    info = ex.info()
    assert info["device_bytes"] < 170 * 10 ** 9, info["device_bytes"]
    sw = info["swap"]
    assert 0.0 <= sw.alpha <= 1.0 and sw.swapped_layers == 2
    assert info["pinned_bytes"] <= sw.cpu_footprint


def test_executor_rejects_bad_configs():
    bad = llama(4, 256, 3, 768, 512, 512)  # head_dim not 64/128
    with pytest.raises(MemoError) as ei:
        Executor(bad, HW, dry_run=1)
    assert ei.value.code == 2
    cp = llama(4, 256, 4, 768, 512, 512)
    cp.sp_or_cp_degree = 2  # SP+TP is tp_degree = t, sp_or_cp_degree = 1
    with pytest.raises(MemoError):
        Executor(cp, HW, dry_run=1)
    # host memory too small for the mandatory offload -> CpuInfeasible (4)
    tiny = P.HardwareConfig(pcie_bandwidth=50e9, cpu_mem=1024, gpu_mem=1 << 40, peak_flops=2.25e15)
    with pytest.raises(MemoError) as ei:
        Executor(CONFIGS["cfg1p"][0], tiny, dry_run=1)
    assert ei.value.code == 4


@pytest.mark.parametrize("t", [2, 4, 8])
def test_tp_rank_plan_bit_exact_and_sized(t):
    """Per-rank SP+TP plan (cfg3 shape scaled down in S): bit-exact with the
    reference planner; skeletal bytes equal the reference model at tp_degree=t."""
    cfg = llama(4, 4096, 32, 11008, 32000, 131072)
    cfg.tp_degree = t
    ex = Executor(cfg, HW, alpha=0.5, dry_run=1)
    trace, plan, info = ex.trace_text(), ex.plan_json(), ex.info()
    assert P.plan_model_json(trace, 0, 60.0, 512) == plan
    if os.path.exists(PROBE):
        assert _ref_plan(trace) == plan
    sz = P.skeletal_sizes(P.ModelConfig(**{**cfg.__dict__, "skeletal_weights": {}}))
    # same weights, per-device bytes shrink by t except the fixed LSE share
    assert info["rb_bytes"] * t == pytest.approx(
        sum(info["skeletal_components"]) * t, rel=0)
    assert info["split"][0] + info["split"][1] == cfg.seq_len


@pytest.mark.parametrize("name,t", [("cfg3_7b_1m", 8), ("cfg4_13b_512k", 2), ("cfg4_13b_512k", 4),
                                    ("cfg4_13b_512k", 8)])
def test_multi_gpu_configs_fit_one_b200_per_rank(name, t):
    """BASELINE configs[2] (7B, 32 layers, S=1M, TP=SP=8) and configs[3] (13B,
    40 layers, S=512K, TP=SP in {2,4,8}) on the paper's node: 2 TiB host shared
    by the t GPUs in use, cpu_mem = 2 TiB / t per GPU (SURVEY §8 HW row,
    discovery 3; this pool's 196 GB host is CpuInfeasible for them, code 4).  Each rank's planned device
    allocation (arena + rounding buffers + bf16 params + f32 grads, one
    cudaMalloc) fits a 180 GB B200; the arena plan is optimal and bit-exact with
    the reference planner; alpha comes from solve_alpha."""
    if name.startswith("cfg3"):
        cfg = llama(32, 4096, 32, 11008, 32000, 1 << 20)
    else:
        cfg = llama(40, 5120, 40, 13824, 32000, 1 << 19)
    cfg.tp_degree = t
    hw = P.HardwareConfig(pcie_bandwidth=50e9, cpu_mem=2048 * P.GiB // t, gpu_mem=180 * 10 ** 9,
                          peak_flops=2.25e15, efficiency=0.5)
    ex = Executor(cfg, hw, dry_run=1, optimizer=0)
    info = ex.info()
    plan = json.loads(ex.plan_json())
    assert plan["optimal"] is True
    assert info["device_bytes"] < 180 * 10 ** 9, (name, t, info["device_bytes"] / 1e9)
    sw = info["swap"]
    assert sw.swapped_layers == cfg.n_layers - 2
    assert 0.0 < sw.alpha <= 1.0
    assert info["pinned_bytes"] <= sw.cpu_footprint <= hw.cpu_mem
    if os.path.exists(PROBE):
        assert _ref_plan(ex.trace_text()) == ex.plan_json()


def test_solo_rank_plan_equals_group_rank_plan_and_option_checks():
    """Communicator kind 4 (one rank measured alone, tools/project_rank.py)
    plans exactly what a rank of the real group plans; the C ABI refuses the
    combinations it cannot honour (CUDA graphs with a multi-rank group, IPC
    handles from a non-IPC communicator) with status 2."""
    from paper_2407_12117_b200.executor import KIND_SOLO
    cfg = llama(4, 4096, 32, 11008, 32000, 131072)
    cfg.tp_degree = 4
    group_rank = Executor(cfg, HW, alpha=0.5, dry_run=1)
    solo = Executor(cfg, HW, alpha=0.5, dry_run=1, tp=(KIND_SOLO, None, 0))
    assert solo.plan_json() == group_rank.plan_json()
    assert solo.info()["device_bytes"] == group_rank.info()["device_bytes"]
    with pytest.raises(MemoError) as e:
        solo.peer_handle()
    assert e.value.code == 2
    with pytest.raises(MemoError) as e:
        Executor(cfg, HW, alpha=0.5, dry_run=1, tp=(KIND_SOLO, None, 0), cuda_graph=1)
    assert e.value.code == 2


def _sizes_of_trace(trace: str):
    sizes = {}
    for line in trace.splitlines():
        parts = line.split()
        if len(parts) == 3 and parts[0] == "malloc":
            sizes[int(parts[1])] = int(parts[2])
    return sizes


def mirror(plan_json: str, trace: str, alignment: int = 512) -> str:
    """Another valid placement of the same trace: every tensor moved to
    total_peak - offset - aligned size.  Disjointness is preserved, so it is a
    legal plan with different addresses."""
    j = json.loads(plan_json)
    peak = j["total_peak"]
    sizes = _sizes_of_trace(trace)
    for a in j["absolute"]:
        sz = -(-sizes[a["tensor"]] // alignment) * alignment
        a["offset"] = peak - a["offset"] - sz
    return json.dumps(j)


def test_bind_plan_accepts_own_reference_and_mirrored_plans():
    """memo_exec_bind_plan: the executor replays a GlobalPlan JSON
    computed outside it -- its own, the reference planner's (oracle/_ref), and a
    different valid placement (mirrored offsets) -- and refuses plans that do
    not fit its trace."""
    cfg, alpha = CONFIGS["cfg1p"]
    ex = Executor(cfg, HW, alpha=alpha, dry_run=1)
    trace, plan = ex.trace_text(), ex.plan_json()
    ex.bind_plan(plan)
    assert ex.plan_json() == plan
    if os.path.exists(PROBE):
        ex.bind_plan(_ref_plan(trace))
        assert ex.plan_json() == plan
    mp = mirror(plan, trace)
    ex.bind_plan(mp)
    assert ex.plan_json() == json.dumps(json.loads(mp), separators=(",", ":"))
    assert ex.plan_json() != plan


def test_bind_plan_refusals():
    cfg, alpha = CONFIGS["cfg1p"]
    ex = Executor(cfg, HW, alpha=alpha, dry_run=1)
    trace, plan = ex.trace_text(), ex.plan_json()
    j = json.loads(plan)

    def code(pj):
        with pytest.raises(MemoError) as e:
            ex.bind_plan(json.dumps(pj) if not isinstance(pj, str) else pj)
        return e.value.code

    assert code("{not json") == 2
    assert code({"total_peak": 0}) == 2
    bad = json.loads(plan)
    bad["absolute"] = bad["absolute"][1:]          # a request left unplaced
    assert code(bad) == 2
    bad = json.loads(plan)
    bad["absolute"].append(dict(bad["absolute"][0], tensor=10 ** 9))   # not in the trace
    assert code(bad) == 2
    bad = json.loads(plan)
    bad["total_peak"] = j["total_peak"] + 512      # more than the reserved arena
    assert code(bad) == 3
    bad = json.loads(plan)
    bad["absolute"][0]["offset"] += 1              # misaligned
    assert code(bad) == 2
    # everything at offset 0: live-together tensors share bytes
    bad = json.loads(plan)
    for a in bad["absolute"]:
        a["offset"] = 0
    assert code(bad) == 2
    ex.bind_plan(plan)                              # still bindable after refusals
