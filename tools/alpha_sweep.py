"""cfg5-style alpha sweep (BASELINE configs[4]) sized to one B200 box: Llama-7B
architecture at 256K tokens with as many layers as the host's pinned memory
allows for the swapped set, alpha in {0, 1/8, ...} up to the host limit.
Reports per alpha: step time, offload/prefetch GB/s (vs the measured pinned
memcpy peak), exposed swap (compute-stream gaps), forward blocking, recompute
time, and measured HBM vs the planned allocation.  Writes one JSON line per alpha.
"""
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from bench import host_link_bandwidth, synthetic_batch  # noqa: E402
from paper_2407_12117_b200 import planner as P  # noqa: E402
from paper_2407_12117_b200._abi import MemoError  # noqa: E402
from paper_2407_12117_b200.executor import Executor  # noqa: E402

S = int(os.environ.get("SWEEP_SEQ", 262144))
N_LAYERS = int(os.environ.get("SWEEP_LAYERS", 6))
STEPS = int(os.environ.get("SWEEP_STEPS", 2))

link = host_link_bandwidth(torch)
host_mem = os.sysconf("SC_PAGE_SIZE") * os.sysconf("SC_PHYS_PAGES")
cfg = P.ModelConfig(n_layers=N_LAYERS, hidden=4096, ffn_hidden=16512, n_heads=32, vocab=32000,
                    seq_len=S, untied_classifier=True)
hw = P.HardwareConfig(pcie_bandwidth=link["d2h"], cpu_mem=int(host_mem * 0.6),
                      gpu_mem=torch.cuda.get_device_properties(0).total_memory, peak_flops=2.25e15)
toks, labels = synthetic_batch(1234, 32000, S)
print(json.dumps({"link": link, "host_mem": host_mem, "seq": S, "layers": N_LAYERS}), flush=True)
for k in range(0, 9, 2):
    alpha = k / 8
    try:
        torch.cuda.synchronize()
        free0, _ = torch.cuda.mem_get_info()
        ex = Executor(cfg, hw, alpha=alpha, optimizer=0, op_timing=0)
        free1, _ = torch.cuda.mem_get_info()
    except MemoError as e:
        print(json.dumps({"alpha": alpha, "skipped": str(e)[:160]}), flush=True)
        if e.code == 4:
            break
        continue
    ex.load_batch(toks, labels)
    ex.step_resident()
    times = []
    for _ in range(STEPS):
        ex.step_resident()
        tl = ex.timeline()
        times.append(ex.info()["last_step_ms"])
    info = ex.info()
    sim = P.simulate(tl, cfg, hw, P.count_params(cfg)["total"])
    off = [e for e in tl if e.kind == "offload"]
    pre = [e for e in tl if e.kind == "prefetch"]
    rec = [e for e in tl if e.kind == "recompute"]
    fwd = [e for e in tl if e.kind == "layer_fwd"]
    off_s = sum(e.end - e.start for e in off)
    pre_s = sum(e.end - e.start for e in pre)
    line = {"alpha": alpha, "split": info["split"], "step_ms": float(np.median(times)),
            "tokens_per_s": S / (np.median(times) * 1e-3),
            "offload_GBps": info["offload_bytes"] / off_s / 1e9 if off_s else None,
            "prefetch_GBps": info["prefetch_bytes"] / pre_s / 1e9 if pre_s else None,
            "link_d2h_GBps": link["d2h"] / 1e9, "link_h2d_GBps": link["h2d"] / 1e9,
            "offload_bytes_per_step": info["offload_bytes"],
            "exposed_swap_s": sim["compute_blocked"], "forward_blocked_s": sim["forward_blocked"],
            "recompute_s": sum(e.end - e.start for e in rec),
            "t_layer_fwd_s": float(np.median([e.end - e.start for e in fwd])),
            "planned_device_bytes": info["device_bytes"], "measured_device_bytes": free0 - free1,
            "pinned_bytes": info["pinned_bytes"],
            "violations": P.validate_schedule(tl, N_LAYERS, info["swap"])}
    print(json.dumps(line), flush=True)
    ex.close()
