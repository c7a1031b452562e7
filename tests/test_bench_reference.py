"""bench.py's reference arm (the CPU implementation of the step) on this host:
one bounded sample, the JSON line's contract, and no import of the product
package on that path (its FLOP model is restated in plain Python)."""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_flop_terms_match_the_planner():
    sys.path.insert(0, ROOT)
    import bench
    from paper_2407_12117_b200 import planner as P
    for name in ("cfg2", "cfg1p", "cfg4s", "cfg5"):
        n, h, H, inter, V, S, _ = bench.CONFIGS[name]
        cfg = P.ModelConfig(n_layers=n, hidden=h, ffn_hidden=inter * 3 // 2, n_heads=H, vocab=V, seq_len=S,
                            untied_classifier=True)
        dense, attn = bench.flop_terms(n, h, H, inter, V, S)
        assert dense + attn == P.estimate_flops_per_sample(cfg, P.count_params(cfg)["total"])


def test_reference_arm_line_without_the_package():
    script = (
        "import sys, json; sys.argv = ['bench.py', '--impl', 'reference', '--steps', '1', '--warmup', '0', "
        "'--config', 'cfg1p']\n"
        "sys.path.insert(0, %r)\n"
        "import bench; bench.main()\n"
        "assert not any(m.startswith('paper_2407_12117_b200') for m in sys.modules), 'product imported'\n" % ROOT)
    out = subprocess.run([sys.executable, "-c", script], capture_output=True, text=True, timeout=600, cwd=ROOT)
    assert out.returncode == 0, out.stderr[-2000:]
    line = json.loads(out.stdout.strip().splitlines()[-1])
    assert line["impl"] == "reference" and line["unit"] == "tokens/s" and line["value"] > 0
    assert line["e2e"] == {"value": line["value"], "unit": "tokens/s", "h2d_bytes_per_step": 0,
                           "d2h_bytes_per_step": 0}
    assert line["cpu_baseline"]["kind"] == "port" and line["cpu_baseline"]["cores"] >= 1
    assert line["config"]["workload"].startswith("tiny 4-layer")
    assert line["ms_per_step"] < 600000  # a measured sample, not the extrapolated workload step
