"""tools/actmem_b200: the reference's `report` (actmem.cpp:227-273) as C++ host
code over the reference's own types, driving libmemo through include/memo.h.
It plans the executor's trace with the reference's actmem::plan_model, binds
that plan (memo_exec_bind_plan), runs real steps and writes cmd_report's
manifest keys with the MEASURED sim and the frag comparison."""
import json
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
DRIVER = os.path.join(ROOT, "tools", "_build", "actmem_b200")

REPORT_KEYS = {"version", "inputs", "model", "hardware", "param_count", "skeletal", "alpha", "plan", "sim", "frag"}
CFG1P = {"model": {"n_layers": 4, "hidden": 256, "ffn_hidden": 1152, "n_heads": 4, "vocab": 512, "batch": 1,
                   "seq_len": 4096, "untied_classifier": True},
         "hardware": {"pcie_bandwidth": 50e9, "cpu_mem": 16 * 2 ** 30, "gpu_mem": 180 * 10 ** 9,
                      "peak_flops": 2.25e15, "efficiency": 0.5}}

needs_driver = pytest.mark.skipif(not os.path.exists(DRIVER), reason="tools/_build/actmem_b200 not built")


@needs_driver
def test_driver_usage_and_bad_input_exit_codes(tmp_path):
    assert subprocess.run([DRIVER], capture_output=True).returncode == 2
    assert subprocess.run([DRIVER, "report", "--config", str(tmp_path / "missing.json")],
                          capture_output=True).returncode == 2
    bad = tmp_path / "bad.json"
    bad.write_text(json.dumps({"model": {"n_layers": 4, "bogus_key": 1}}))
    assert subprocess.run([DRIVER, "report", "--config", str(bad)], capture_output=True).returncode == 2


@pytest.mark.gpu
@needs_driver
def test_driver_report_cfg1p(tmp_path):
    cfg = tmp_path / "cfg1p.json"
    cfg.write_text(json.dumps(CFG1P))
    out, tl = tmp_path / "manifest.json", tmp_path / "timeline.csv"
    r = subprocess.run([DRIVER, "report", "--config", str(cfg), "--alpha", "0.5", "--steps", "3", "--out", str(out),
                        "--timeline", str(tl)], capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stderr
    m = json.loads(out.read_text())
    assert REPORT_KEYS <= set(m)
    assert m["plan"]["optimal"] is True and m["plan"]["total_peak"] == m["measured"]["arena_bytes"]
    assert m["alpha"]["alpha"] == 0.5 and m["measured"]["swap_tokens"] == 2048
    assert m["measured"]["schedule_violations"] == []
    assert m["sim"]["iteration_time"] > 0 and m["sim"]["mfu"] > 0
    assert m["frag"]["planned"]["peak_reserved"] == m["plan"]["total_peak"]
    losses = m["measured"]["losses"]
    assert len(losses) == 3 and all(5.0 < x < 8.0 for x in losses)
    assert tl.read_text().startswith("stream,kind,layer,start,end")
