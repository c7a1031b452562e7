"""Summarise ncu captures (gpurun_out/prof_*.ncu-rep, launches.csv) into
profiles/ncu_summary.json + a markdown table.  Run here (no GPU needed):
    python tools/ncu_summary.py gpurun_out profiles/ncu_r01
"""
import csv
import io
import json
import os
import subprocess
import sys
from collections import defaultdict

METRICS = {
    "gpu__time_duration.sum": "duration_ns",
    "dram__bytes_read.sum": "dram_read",
    "dram__bytes_write.sum": "dram_write",
    "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active": "tensor_pipe_pct",
    "sm__inst_executed_pipe_tensor.avg.pct_of_peak_sustained_active": "tensor_inst_pct",
    "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed": "dram_pct",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed": "sm_pct",
    "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed": "smem_pct",
    "sm__warps_active.avg.pct_of_peak_sustained_active": "warps_active_pct",
    "launch__registers_per_thread": "regs",
    "sm__cycles_elapsed.avg.per_second": "sm_hz",
    "sm__pipe_xu_cycles_active.avg.pct_of_peak_sustained_active": "xu_pipe_pct",
    "smsp__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active": "xu_inst_pct",
    "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active": "fma_pipe_pct",
    "sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active": "alu_pipe_pct",
    "lts__throughput.avg.pct_of_peak_sustained_elapsed": "l2_pct",
    "sm__pipe_tc_cycles_active.avg.pct_of_peak_sustained_active": "tc_pipe_pct",
    "sm__issue_active.avg.pct_of_peak_sustained_active": "issue_pct",
}


def raw(rep):
    out = subprocess.check_output(["ncu", "-i", rep, "--page", "raw", "--csv"], text=True)
    rows = list(csv.reader(io.StringIO(out)))
    hdr = rows[0]
    res = []
    for r in rows[2:]:
        d = dict(zip(hdr, r))
        item = {"kernel": d.get("Kernel Name", "")[:80]}
        for m, k in METRICS.items():
            if m in d:
                try:
                    item[k] = float(d[m].replace(",", ""))
                except ValueError:
                    item[k] = d[m]
        res.append(item)
    return res


def launches(path):
    per = defaultdict(lambda: [0, 0.0])
    with open(path) as f:
        lines = [l for l in f if l.startswith('"')]
    rd = csv.DictReader(io.StringIO("".join(lines)))
    for r in rd:
        if r.get("Metric Name") != "gpu__time_duration.sum":
            continue
        name = r["Kernel Name"].split("(")[0].split("<")[0][:60]
        v = float(r["Metric Value"].replace(",", ""))
        unit = r.get("Metric Unit", "ns")
        ns = v * {"ns": 1, "usecond": 1e3, "us": 1e3, "msecond": 1e6, "ms": 1e6, "second": 1e9}.get(unit, 1)
        per[name][0] += 1
        per[name][1] += ns
    tot = sum(v[1] for v in per.values())
    return {k: {"launches": v[0], "total_ms": v[1] / 1e6, "share": v[1] / tot}
            for k, v in sorted(per.items(), key=lambda kv: -kv[1][1])}


def main():
    src, dst = sys.argv[1], sys.argv[2]
    summary = {}
    for f in sorted(os.listdir(src)):
        if f.startswith("prof_") and f.endswith(".ncu-rep"):
            try:
                summary[f[5:-8]] = raw(os.path.join(src, f))
            except subprocess.CalledProcessError as e:
                summary[f[5:-8]] = {"error": str(e)}
    if os.path.exists(os.path.join(src, "launches.csv")):
        summary["launch_list"] = launches(os.path.join(src, "launches.csv"))
    with open(dst + ".json", "w") as f:
        json.dump(summary, f, indent=1)
    print(json.dumps(summary, indent=1)[:6000])


if __name__ == "__main__":
    main()
