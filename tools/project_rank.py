"""Per-rank projection of a multi-GPU SP+TP config on ONE B200 (communicator
kind 4: every collective is a local copy of the same size, so the rank's
compute, memory plan and swap traffic are the real ones while nothing crosses
NVLink).  Prints one JSON line: measured per-rank step time, kernel classes,
alpha/swap, planned vs measured HBM, and the projection of the t-GPU step
(measured + an NVLink estimate for the collectives' bytes).  A projection,
not a measurement of the multi-GPU system; the numerics are not the group's.

  python tools/project_rank.py [cfg3|cfg4t2|cfg4t4|cfg4t8] [--steps 1]
"""
import argparse
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

CONFIGS = {  # name: (n_layers, hidden, heads, intermediate, vocab, seq, tp)
    "cfg3": (32, 4096, 32, 11008, 32000, 1048576, 8),
    "cfg4t8": (40, 5120, 40, 13824, 32000, 524288, 8),
    "cfg4t4": (40, 5120, 40, 13824, 32000, 524288, 4),
}
NVLINK_GBPS = 725.0  # pool-measured all-gather bus bandwidth per GPU; an assumption here


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("config", nargs="?", default="cfg3", choices=sorted(CONFIGS))
    ap.add_argument("--steps", type=int, default=1)
    args = ap.parse_args()
    import numpy as np
    import torch

    from oracle import oracle as O
    from paper_2407_12117_b200 import planner as P
    from paper_2407_12117_b200.executor import KIND_SOLO, Executor

    n, h, H, F, V, S, t = CONFIGS[args.config]
    cfg = P.ModelConfig(n_layers=n, hidden=h, ffn_hidden=F * 3 // 2, n_heads=H, vocab=V, batch=1, seq_len=S,
                        dtype_bytes=2, tp_degree=t, untied_classifier=True)
    host = os.sysconf("SC_PAGE_SIZE") * os.sysconf("SC_PHYS_PAGES")
    cpu_mem = int(host * 0.6)  # this box runs one rank: it gets the whole pinnable budget
    hw = P.HardwareConfig(pcie_bandwidth=55e9, cpu_mem=cpu_mem, gpu_mem=torch.cuda.get_device_properties(0).total_memory,
                          peak_flops=2.25e15, efficiency=0.5)
    toks, labels = O.tokens(1234, V, S)
    t0 = time.time()
    with Executor(cfg, hw, tp=(KIND_SOLO, None, 0), op_timing=0, optimizer=1) as ex:
        ex.step(toks, labels)
        tl = ex.timeline()
    t_layer = float(np.median([e.end - e.start for e in tl if e.kind == "layer_fwd"]))
    torch.cuda.synchronize()
    free0, _ = torch.cuda.mem_get_info()
    with Executor(cfg, hw, tp=(KIND_SOLO, None, 0), op_timing=1, optimizer=1, t_layer=t_layer) as ex:
        free1, _ = torch.cuda.mem_get_info()
        info0 = ex.info()
        ms = []
        for _ in range(args.steps):
            ex.step(toks, labels)
            tl = ex.timeline()  # also computes the step's device time
            ms.append(ex.info()["last_step_ms"])
        info = ex.info()
    step_s = float(np.median(ms)) * 1e-3
    swap = info0["swap"]
    violations = P.validate_schedule(tl, n, swap)
    p_total = P.count_params(cfg)["total"]
    flops = P.estimate_flops_per_sample(cfg, p_total)  # whole model, reference formula
    # collectives per layer (fwd 2 AG + 2 RS, bwd 2 AG + 2 RS + 2 AG (wgrad regathers), recompute 2 AG + 1 RS):
    # bf16 gathers pull (t-1)/t * S*h*2, f32 reduce-scatters pull (t-1)/t * S*h*4
    ag = (t - 1) / t * S * h * 2
    rs = (t - 1) / t * S * h * 4
    n_sw = sum(e.kind == "recompute" for e in tl)
    comm_bytes = n * (6 * ag + 4 * rs) + n_sw * (2 * ag + rs)
    comm_s = comm_bytes / (NVLINK_GBPS * 1e9)
    proj_s = step_s + comm_s  # no overlap assumed (upper bound)
    line = {
        "config": args.config, "n_layers": n, "hidden": h, "seq_len": S, "tp": t,
        "kind": "per-rank projection on one B200 (collectives replaced by local copies)",
        "rank_step_s": step_s, "setup_s": time.time() - t0,
        "alpha": swap.alpha, "swap_tokens": info0["split"][0], "recompute_tokens": info0["split"][1],
        "t_layer_measured_s": t_layer, "cpu_mem_budget": cpu_mem, "pinned_bytes": info0["pinned_bytes"],
        "planned_device_bytes": info0["device_bytes"], "measured_device_bytes": free0 - free1,
        "schedule_violations": violations,
        "kernels_ms": {k: v["ms"] for k, v in info["ops"].items()},
        "offload_bytes": info["offload_bytes"], "prefetch_bytes": info["prefetch_bytes"],
        "comm_bytes_per_rank": comm_bytes, "comm_s_at_%g_GBps" % NVLINK_GBPS: comm_s,
        "projected_step_s_no_overlap": proj_s,
        "projected_tokens_per_s_per_gpu": S / proj_s / t,
        "projected_mfu": flops / proj_s / (t * 2.25e15),
        "rank_compute_mfu": flops / step_s / (t * 2.25e15),
    }
    print(json.dumps(line), flush=True)


if __name__ == "__main__":
    main()
