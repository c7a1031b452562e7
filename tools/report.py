"""`report`-style run manifest on real hardware (the analogue of
actmem.cpp:227-273 cmd_report): config + FNV input hashes (json_io.hpp:265), the
executor's trace/plan hashes, swap plan, token split, the MEASURED schedule as
the reference's timeline CSV (json_io.hpp:246) and its SimReport, plus measured
HBM vs the planned allocation.  `--dry-run` works without a GPU (plan only).

  python tools/report.py --config cfg1p [--dry-run] [--out manifest.json] [--timeline t.csv]
"""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from bench import CONFIGS, synthetic_batch  # noqa: E402
from paper_2407_12117_b200 import _abi  # noqa: E402
from paper_2407_12117_b200 import planner as P  # noqa: E402
from paper_2407_12117_b200.executor import Executor  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="cfg1p", choices=sorted(CONFIGS))
    ap.add_argument("--alpha", type=float, default=-1.0)
    ap.add_argument("--dry-run", action="store_true")
    ap.add_argument("--out")
    ap.add_argument("--timeline")
    a = ap.parse_args()
    n, h, H, inter, V, S, desc = CONFIGS[a.config]
    cfg = P.ModelConfig(n_layers=n, hidden=h, ffn_hidden=inter * 3 // 2, n_heads=H, vocab=V,
                        seq_len=S, untied_classifier=True)
    hw = P.HardwareConfig(pcie_bandwidth=50e9, cpu_mem=96 * P.GiB, gpu_mem=180 * 10 ** 9,
                          peak_flops=2.25e15)
    config_json = json.dumps({"model": cfg.to_json(), "hardware": hw.__dict__}, sort_keys=True)
    ex = Executor(cfg, hw, alpha=a.alpha, dry_run=int(a.dry_run), optimizer=0)
    info = ex.info()
    trace, plan = ex.trace_text(), ex.plan_json()
    sw = info["swap"]
    man = {"version": _abi.lib.memo_version().decode(), "workload": desc,
           "inputs": {"config_fnv": P.fnv1a_hex(config_json), "trace_fnv": P.fnv1a_hex(trace)},
           "plan": {"plan_fnv": P.fnv1a_hex(plan), "total_peak": json.loads(plan)["total_peak"],
                    "optimal": json.loads(plan)["optimal"]},
           "swap": {"alpha": sw.alpha, "mandatory_bytes": sw.mandatory_bytes,
                    "swapped_bytes_per_layer": sw.swapped_bytes_per_layer,
                    "cpu_footprint": sw.cpu_footprint, "swapped_layers": sw.swapped_layers,
                    "blocking": None if sw.mandatory_stall is None else {"stall_seconds": sw.mandatory_stall}},
           "token_split": {"swap_tokens": info["split"][0], "recompute_tokens": info["split"][1]},
           "memory": {k: info[k] for k in ("arena_bytes", "rb_bytes", "state_bytes", "device_bytes",
                                             "pinned_bytes")}}
    if not a.dry_run:
        import torch
        toks, labels = synthetic_batch(1234, V, S)
        ex.step(toks, labels)
        events = ex.timeline()
        man["loss"] = ex.loss()
        man["sim"] = P.simulate(events, cfg, hw, P.count_params(cfg)["total"])
        man["schedule_violations"] = P.validate_schedule(events, n, sw)
        csv = P.schedule_timeline_csv(events)
        man["timeline_fnv"] = P.fnv1a_hex(csv)
        if a.timeline:
            with open(a.timeline, "w") as f:
                f.write(csv)
        free, total = torch.cuda.mem_get_info()
        man["memory"]["device_used_after_step"] = total - free
    ex.close()
    text = json.dumps(man, indent=1)
    if a.out:
        with open(a.out, "w") as f:
            f.write(text + "\n")
    print(text)


if __name__ == "__main__":
    main()
